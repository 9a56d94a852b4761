# Round evidence: gpu tests, smoke, default bench, reference arm, ncu launch list.
# usage: bash scripts/gpu_evidence.sh TAG   (one ncu tool per call; full capture: gpu_ncu_full.sh)
set -x
TAG=${1:-r01}
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gpu_tests_$TAG.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference_$TAG.log 2>&1; echo ref_rc=$?
SMALL="bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-powersgd --secondary none"
timeout 300 python $SMALL > gpurun_out/bench_small_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python $SMALL > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu1_rc=$?
