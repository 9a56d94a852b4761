# Balance check: per-kernel SM-active average vs max (ncu), all our kernels of one P+Q pair
W=${1:-resnet50-r4}
T=${2:-bal}
SMALL="bench.py --workload $W --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-powersgd --secondary none"
timeout 300 python $SMALL > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max,gpc__cycles_elapsed.max,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/$T.csv -k regex:"stream_kernel|row_kernel|orth_kernel|col_reduce|tc_kernel" python $SMALL > gpurun_out/ncu_bal.log 2>&1; echo ncu_rc=$?
