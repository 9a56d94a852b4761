# ncu --set full of one K1-P (mode 0) and one K1-Q (mode 3) launch of a workload.
# usage: bash scripts/gpu_ncu_k1p_w.sh WORKLOAD [TAG]
W=${1:-bert-large-r4}
T=${2:-$W}
SMALL="bench.py --workload $W --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-powersgd --secondary none"
timeout 300 python $SMALL > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"stream_kernel<.int.[03]" -s 2 -c 2 -o gpurun_out/prof_k1_$T python $SMALL > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
