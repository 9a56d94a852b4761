# Round-2 multi-GPU evidence on one N-GPU box (raw logs under gpurun_out/mg_*):
#  1. parity: tests/mgpu_check.py (NCCL, bucket policies, bucket API, Power-SGD,
#     NVLS separate + fused, tensor-core path r=8 with NCCL and fused NVLS)
#  2. bench lines at N: BERT-L r=4 / r=32, ResNet-50 r=4, NCCL vs NVLS (+ S-SGD)
#  3. ResNet-152 tensor-fusion buffer sweep (BASELINE configs[2]):
#     default_bucket_bytes in {0, 1, 5, 25, 100 MiB, single} x {nccl, nvls}
# usage: bash scripts/gpu_multi_r02.sh N
N=${1:-2}
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/mg_build.log 2>&1
nvidia-smi topo -m > gpurun_out/mg_topo_$N.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29533 tests/mgpu_check.py > gpurun_out/mg_parity_$N.log 2>&1; echo mgpu_rc=$?
grep -E "^run|mgpu ok|Error|error" gpurun_out/mg_parity_$N.log | tail -12
summ() {
python - "$1" <<'PY'
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
    ss = d.get("ssgd") or {}
    print(sys.argv[1].split("/")[-1], "ms", round(d["ms_per_step"], 4), "GB/s", round(d["value"], 1), "ar", d["config"]["allreduce"],
          "buckets", d["config"].get("buckets_PQ"), "P/Q", round(d["step_stats"]["p_step_ms"], 4), round(d["step_stats"]["q_step_ms"], 4),
          "nvlink", d.get("nvlink"), "ssgd_ms", ss.get("ms_per_step"))
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
}
P=29600
for W in bert-large-r4 resnet50-r4 bert-large-r32; do
  for AR in nccl nvls; do
    P=$((P + 1))
    EXTRA="--no-ssgd"; [ $W = bert-large-r4 ] && [ $AR = nccl ] && EXTRA=""
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --workload $W --steps 30 --warmup 5 --no-e2e --no-powersgd $EXTRA --secondary none --allreduce $AR > gpurun_out/mg_bench_${N}_${W}_$AR.log 2>&1
    summ gpurun_out/mg_bench_${N}_${W}_$AR.log
  done
done
[ -n "$NO_SWEEP" ] && exit 0
for BB in 0 1048576 5242880 26214400 104857600 -1; do
  for AR in nccl nvls; do
    P=$((P + 1))
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --workload resnet152-r4 --bucket-bytes $BB --steps 30 --warmup 5 --no-e2e --no-powersgd --no-ssgd --secondary none --allreduce $AR > gpurun_out/mg_sweep_${N}_${BB}_$AR.log 2>&1
    summ gpurun_out/mg_sweep_${N}_${BB}_$AR.log
  done
done
