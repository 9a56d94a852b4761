W=${1:-bert-large-r4}
python bench.py --workload $W --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --secondary none > gpurun_out/bench_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"stream_kernel<.int.0" -s 1 -c 1 -o gpurun_out/prof_k1p_$W python bench.py --workload $W --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --secondary none > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
