# col_reduce batched slot loads + K2 grid capped at the busy items: tests + A/B vs lib/libacp_base.so
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_ovh.log 2>&1 || { cat gpurun_out/build_ovh.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_determinism.py tests/test_gpu_fullsize.py tests/test_gpu_tc.py -m gpu -x -q > gpurun_out/ovh_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/ovh_tests.log
VARIANTS="base new" timeout 900 bash scripts/gpu_abn.sh ${@:-resnet50-r4 resnet152-r4 bert-large-r4 bert-base-r8}
