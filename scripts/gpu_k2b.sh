mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_k2.log 2>&1 || { cat gpurun_out/build_k2.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_edge.py tests/test_gpu_parity.py -m gpu -x -q -k "16 or 32 or degenerate or ill or ragged or cfg1" > gpurun_out/k2_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/k2_tests.log
VARIANTS="base new" timeout 900 bash scripts/gpu_abn.sh bert-large-r4 bert-large-r16 bert-large-r32 resnet50-r4 2>&1 | head -8
