# adaptive per-segment cost in the SIMT work split: tests + A/B against lib/libacp_base.so
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_seg.log 2>&1 || { cat gpurun_out/build_seg.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_determinism.py -m gpu -x -q -k "not 32 and not 16 and not 8" > gpurun_out/seg_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/seg_tests.log
VARIANTS="base new" timeout 900 bash scripts/gpu_abn.sh ${@:-bert-large-r4 resnet50-r4 resnet152-r4 bert-large-r1}
