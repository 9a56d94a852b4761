python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --secondary none > gpurun_out/bench_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stream_kernel" -s 2 -c 4 -o gpurun_out/prof_stream3 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --secondary none > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
