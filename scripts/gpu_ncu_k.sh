# ncu --set full of selected kernels of one workload (after the plain run exits 0)
# usage: KREGEX=... SKIP=.. COUNT=.. bash scripts/gpu_ncu_k.sh WORKLOAD TAG
W=${1:-bert-large-r8}
T=${2:-k}
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_$T.log 2>&1
SMALL="bench.py --workload $W --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-powersgd --secondary none"
timeout 300 python $SMALL > gpurun_out/bench_small_$T.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"${KREGEX:-tc5}" -s ${SKIP:-2} -c ${COUNT:-2} -o gpurun_out/prof_$T python $SMALL > gpurun_out/ncu_$T.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/ncu_$T.log
