mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_k1.log 2>&1 || { cat gpurun_out/build_k1.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_edge.py tests/test_gpu_parity.py -m gpu -x -q -k "tc or 8 or 16 or 32" > gpurun_out/k1_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/k1_tests.log; grep -m3 -E "Error|error|rel err" gpurun_out/k1_tests.log
VARIANTS="new:ACP_NO_TC5K1=1 new" timeout 900 bash scripts/gpu_abn.sh bert-large-r8 bert-large-r32 bert-base-r8 2>&1 | head -6
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "32 or 8" > gpurun_out/k1_full.log 2>&1; echo full_rc=$?; tail -3 gpurun_out/k1_full.log
