# Round-2 evidence on one B200 for the current tree (TAG): GPU tests (with
# durations), smoke, the default bench line, the reference arm, the ncu
# launch list, one `ncu --set full` capture per workload (-> traffic json
# tagged with the build id), and the per-workload sweep.
# usage: bash scripts/gpu_evidence_r02.sh TAG
set -x
TAG=${1:-r02}
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_$TAG.log 2>&1 || { cat gpurun_out/build_$TAG.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=25 > gpurun_out/gpu_tests_$TAG.log 2>&1; echo tests_rc=$?; tail -4 gpurun_out/gpu_tests_$TAG.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke_$TAG.log
# ncu --set full captures first (the traffic json must exist before the bench line reads it)
rm -f gpurun_out/*.ncu-rep
for W in bert-large-r4 resnet50-r4 bert-large-r32 bert-large-r8; do
  SMALL="bench.py --workload $W --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-powersgd --secondary none"
  timeout 300 python $SMALL > gpurun_out/bench_small_${TAG}_$W.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"stream_kernel|k1p_kernel|row_kernel|orth_kernel|col_reduce|tc_kernel|tc5_" -s 8 -c 9 -o gpurun_out/prof_${TAG}_$W python $SMALL > gpurun_out/ncu_full_${TAG}_$W.log 2>&1; echo ncu_${W}_rc=$?
  python scripts/traffic_from_ncu.py gpurun_out/prof_${TAG}_$W.ncu-rep $W $TAG
  python scripts/summarize_ncu.py full gpurun_out/prof_${TAG}_$W.ncu-rep gpurun_out/${TAG}_ncu_full_$W.md > /dev/null
  # only gpurun_out/ comes back (<= 64 MiB): keep the json and the summaries
  cp profiles/ncu_traffic_$TAG.json gpurun_out/ 2>/dev/null; rm -f gpurun_out/prof_${TAG}_$W.ncu-rep
done
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1; echo bench_rc=$?; tail -c 400 gpurun_out/bench_default_$TAG.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference_$TAG.log 2>&1; echo ref_rc=$?
SMALL="bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-powersgd --secondary none"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python $SMALL > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu1_rc=$?
python scripts/summarize_ncu.py launches gpurun_out/launches_$TAG.csv gpurun_out/${TAG}_launches.md > /dev/null
bash scripts/gpu_sweep_all.sh ${TAG}_sweep > /dev/null 2>&1; echo sweep_rc=$?
