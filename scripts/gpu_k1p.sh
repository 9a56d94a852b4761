mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_k1p.log 2>&1 || { cat gpurun_out/build_k1p.log; exit 1; }
ACP_K1P_SPLIT=1 ACP_STREAM_BUDGET_KB=216 timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_edge.py -m gpu -x -q -k "bert-large-4-None or ragged or medium or resnet50" > gpurun_out/k1p_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/k1p_tests.log
VARIANTS="new new:ACP_STREAM_BUDGET_KB=216 new:ACP_K1P_SPLIT=1,ACP_STREAM_BUDGET_KB=216 new:ACP_K1P_SPLIT=1,ACP_STREAM_BUDGET_KB=216,ACP_K1P_WIDE_TT=8192 new:ACP_K1P_SPLIT=1,ACP_STREAM_BUDGET_KB=200" timeout 900 bash scripts/gpu_abn.sh bert-large-r4 resnet50-r4 2>&1 | head -10
