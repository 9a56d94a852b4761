# GPU test suite with per-test durations, smoke, and the default bench line.
# usage: bash scripts/gpu_tests.sh TAG [pytest -k expr]
set -x
TAG=${1:-r02}
K=${2:-}
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_$TAG.log 2>&1
if [ -n "$K" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -rs --durations=0 -k "$K" > gpurun_out/gpu_tests_$TAG.log 2>&1; echo tests_rc=$?
else
  timeout 2400 python -m pytest tests -m gpu -q -rs --durations=0 > gpurun_out/gpu_tests_$TAG.log 2>&1; echo tests_rc=$?
fi
tail -40 gpurun_out/gpu_tests_$TAG.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1; echo bench_rc=$?; tail -c 600 gpurun_out/bench_default_$TAG.log
