mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_tc5.log 2>&1 || { cat gpurun_out/build_tc5.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_edge.py -m gpu -x -q -k "tc or 8 or 32" > gpurun_out/tc5_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/tc5_tests.log
VARIANTS="new:ACP_NO_TC5=1 new" timeout 900 bash scripts/gpu_abn.sh bert-large-r8 bert-large-r16 bert-large-r32 bert-base-r8 2>&1 | head -8
