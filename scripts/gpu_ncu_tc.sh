# ncu --set full of the four TC kernels (K1-P, K1-Q, decode P, decode Q) of one P+Q step pair
# usage: bash scripts/gpu_ncu_tc.sh WORKLOAD TAG
W=${1:-bert-large-r8}
T=${2:-tc}
SMALL="bench.py --workload $W --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-powersgd --secondary none"
timeout 300 python $SMALL > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"${KREGEX:-tc_kernel}" -s ${SKIP:-4} -c ${COUNT:-4} -o gpurun_out/prof_$T python $SMALL > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
