timeout 900 python -m pytest tests -m gpu -x -q -k "ragged or cfg1" > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gpu_tests.log
for W in bert-large-r8 bert-base-r8; do
  timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --secondary none > gpurun_out/sweep_$W.log 2>&1; echo $W rc=$?
done
