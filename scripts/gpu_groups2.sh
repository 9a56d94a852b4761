# N-GPU compute-group sweep (ACP_COMPUTE_GROUPS) for ResNet-50 and BERT-L
N=${1:-2}
for G in 1 2 4; do
  for W in resnet50-r4 bert-large-r4; do
    ACP_COMPUTE_GROUPS=$G timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 100)) bench.py --gpus $N --workload $W --steps 30 --warmup 5 --no-e2e --no-powersgd --no-ssgd --secondary none > gpurun_out/cg_${N}_${G}_$W.log 2>&1
    python - $N $G $W <<'PY'
import json, sys
try:
    d = json.loads([l for l in open(f"gpurun_out/cg_{sys.argv[1]}_{sys.argv[2]}_{sys.argv[3]}.log") if l.startswith("{")][-1])
    print(sys.argv[1], "groups", sys.argv[2], sys.argv[3], "ms", round(d["ms_per_step"], 4))
except Exception as e:
    print(sys.argv[1:], "FAILED", e)
PY
  done
done
