# K2 thread-per-row apply at r >= 16, Power-SGD at r = 16 / 32, determinism test:
# GPU tests, then A/B against the HEAD build (lib/libacp_base.so)
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_k2r32.log 2>&1 || { cat gpurun_out/build_k2r32.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_powersgd.py tests/test_gpu_determinism.py tests/test_gpu_edge.py tests/test_gpu_parity.py tests/test_gpu_tc.py -m gpu -x -q > gpurun_out/k2r32_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/k2r32_tests.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "32 or bert-base" > gpurun_out/k2r32_full.log 2>&1; echo full_rc=$?; tail -2 gpurun_out/k2r32_full.log
VARIANTS="base new" timeout 900 bash scripts/gpu_abn.sh ${@:-bert-large-r32 bert-large-r16}
for W in bert-large-r32 bert-large-r16; do timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --secondary none > gpurun_out/psgd_$W.log 2>&1; python -c "
import json,sys; d=json.loads(open('gpurun_out/psgd_$W.log').read().strip().splitlines()[-1]); print('$W', 'acp', round(d['ms_per_step'],4), 'psgd', d['powersgd'])"; done
