set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.log 2>&1; echo ref_rc=$?
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --secondary none > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01_v2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --secondary none > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"stream_kernel|row_kernel|orth_kernel|col_reduce" -s 8 -c 9 -o gpurun_out/prof_r01_v2 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --secondary none > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
