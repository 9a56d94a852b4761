# two-row K1-P' (k1p_kernel): parity tests at r <= 4, then A/B against seg_k1p (ACP_K1P_OLD=1)
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_k1p2.log 2>&1 || { cat gpurun_out/build_k1p2.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py -m gpu -x -q -k "not 8 and not 16 and not 32" > gpurun_out/k1p2_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/k1p2_tests.log
VARIANTS="new:ACP_K1P_OLD=1 new" timeout 900 bash scripts/gpu_abn.sh ${@:-bert-large-r4 resnet50-r4 bert-large-r1 resnet152-r4}
