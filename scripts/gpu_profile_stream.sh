set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
tail -5 gpurun_out/gpu_tests.log
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --secondary none > gpurun_out/bench_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stream_kernel" -s 6 -c 3 -o gpurun_out/prof_stream python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --secondary none > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
