# K2 register Cholesky (r >= 16) with rsqrt / reciprocal products: tests + A/B vs lib/libacp_base.so
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_chol32.log 2>&1 || { cat gpurun_out/build_chol32.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py tests/test_gpu_tc.py tests/test_gpu_determinism.py tests/test_gpu_fullsize.py tests/test_gpu_powersgd.py -m gpu -x -q -k "16 or 32 or ill or degenerate" > gpurun_out/chol32_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/chol32_tests.log
VARIANTS="base new" timeout 900 bash scripts/gpu_abn.sh ${@:-bert-large-r32 bert-large-r16}
