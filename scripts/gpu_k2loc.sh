# K2 whole-factor-in-one-CTA path (orth_local): GPU tests, then A/B against ACP_ORTH_LOCAL=0
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_k2loc.log 2>&1 || { cat gpurun_out/build_k2loc.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/k2loc_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/k2loc_tests.log
VARIANTS="new:ACP_ORTH_LOCAL=0 new" timeout 900 bash scripts/gpu_abn.sh ${@:-resnet50-r4 bert-large-r4 resnet152-r4 bert-base-r8}
