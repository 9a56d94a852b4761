# N-GPU bench: NCCL vs NVLS all-reduce for BERT-L r=4 and ResNet-50 r=4
N=${1:-2}
for AR in nccl nvls; do
  for W in bert-large-r4 resnet50-r4; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port $((29580 + RANDOM % 100)) bench.py --gpus $N --workload $W --steps 30 --warmup 5 --no-e2e --no-powersgd --no-ssgd --secondary none --allreduce $AR > gpurun_out/nv_${N}_${AR}_$W.log 2>&1
    python - $N $AR $W <<'PY'
import json, sys
try:
    d = json.loads([l for l in open(f"gpurun_out/nv_{sys.argv[1]}_{sys.argv[2]}_{sys.argv[3]}.log") if l.startswith("{")][-1])
    print(sys.argv[1], sys.argv[2], sys.argv[3], "ms", round(d["ms_per_step"], 4), "ar", d["config"]["allreduce"], "P/Q", round(d["step_stats"]["p_step_ms"], 4), round(d["step_stats"]["q_step_ms"], 4), "nvlink", d["nvlink"])
except Exception as e:
    print(sys.argv[1:], "FAILED", e)
PY
  done
done
