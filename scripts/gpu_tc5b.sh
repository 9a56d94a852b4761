set -x
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_tc5.log 2>&1 || { cat gpurun_out/build_tc5.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_tc.py -m gpu -x -q > gpurun_out/tc5_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/tc5_tests.log
VARIANTS="new:ACP_NO_TC5=1 new" timeout 900 bash scripts/gpu_abn.sh bert-large-r8 bert-large-r32 bert-base-r8 2>&1 | head -6
KREGEX=tc5 SKIP=2 COUNT=2 bash scripts/gpu_ncu_k.sh bert-base-r8 ${TAG:-tc5b}
