set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench1.log 2>&1; echo bench_rc=$?
tail -c 3000 gpurun_out/bench1.log
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --secondary none > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --secondary none > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"row_kernel|col_kernel|orth_kernel" -s 12 -c 8 -o gpurun_out/prof_r01 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --secondary none > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
ls -la gpurun_out
