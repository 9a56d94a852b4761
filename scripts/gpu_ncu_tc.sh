# ncu --set full of one TC P-step and one TC Q-step K1 launch (+ parity tests first)
# usage: bash scripts/gpu_ncu_tc.sh WORKLOAD TAG
W=${1:-bert-large-r4}
T=${2:-tc}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/tc_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/tc_tests.log
SMALL="bench.py --workload $W --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-powersgd --secondary none"
timeout 300 python $SMALL > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"tc_kernel" -s 2 -c 2 -o gpurun_out/prof_$T python $SMALL > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
