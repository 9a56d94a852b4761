mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_pf.log 2>&1 || { cat gpurun_out/build_pf.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_edge.py -m gpu -x -q -k "tc or 4 or 8 or 32" > gpurun_out/pf_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/pf_tests.log
VARIANTS="new:ACP_NO_TC5K1=1 new" timeout 900 bash scripts/gpu_abn.sh bert-large-r8 bert-large-r32 bert-base-r8 2>&1 | head -6

