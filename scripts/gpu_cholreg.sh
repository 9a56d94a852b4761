# K2 whole-factor items with the register Cholesky: tests + A/B vs lib/libacp_base.so
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_cr.log 2>&1 || { cat gpurun_out/build_cr.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_fullsize.py -m gpu -x -q -k "not 32" > gpurun_out/cr_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/cr_tests.log
VARIANTS="base new" timeout 900 bash scripts/gpu_abn.sh ${@:-resnet50-r4 resnet152-r4 bert-large-r4 bert-base-r8}
