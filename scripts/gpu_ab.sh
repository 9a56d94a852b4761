# Quick A/B: GPU parity tests, then per-kernel-class times for the given workloads.
# usage: bash scripts/gpu_ab.sh [workload ...]
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/ab_tests.log
for W in ${@:-bert-large-r4 resnet50-r4}; do
  timeout 300 python bench.py --workload $W --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-powersgd --secondary none > gpurun_out/ab_$W.log 2>&1
  python - "$W" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.log").read().strip().splitlines()[-1])
    pc = d["roofline"]["per_class"]
    print(sys.argv[1], "ms/step %.4f" % d["ms_per_step"], " ".join("%s=%.4fms/%.0fGB/s" % (k, v["ms_per_launch"], v["gbs"]) for k, v in pc.items()))
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
