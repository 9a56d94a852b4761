# ncu --set full (source counters) of ONE deferred K1-P' launch (BERT-L r=4),
# kept as a single-kernel report small enough to come back in gpurun_out/
T=${1:-k1p}
W=${2:-bert-large-r4}
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_$T.log 2>&1 || exit 1
SMALL="bench.py --workload $W --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-powersgd --secondary none"
timeout 300 python $SMALL > gpurun_out/bench_small_$T.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"${KREGEX:-stream_kernel<.int.0}" -s ${SKIP:-1} -c 1 -o gpurun_out/prof_$T python $SMALL > gpurun_out/ncu_$T.log 2>&1; echo ncu_rc=$?
ls -la gpurun_out/prof_$T.ncu-rep
