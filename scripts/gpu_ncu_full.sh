# One ncu --set full capture of every kernel class of one ACP P+Q step pair.
# usage: bash scripts/gpu_ncu_full.sh TAG [WORKLOAD]
set -x
TAG=${1:-r01}
W=${2:-bert-large-r4}
SMALL="bench.py --workload $W --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-powersgd --secondary none"
timeout 300 python $SMALL > gpurun_out/bench_small_$TAG.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"stream_kernel|row_kernel|orth_kernel|col_reduce" -s 8 -c 9 -o gpurun_out/prof_$TAG python $SMALL > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu2_rc=$?
