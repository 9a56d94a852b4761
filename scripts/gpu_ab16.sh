mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_ab16.log 2>&1 || { cat gpurun_out/build_ab16.log; exit 1; }
VARIANTS="new:ACP_NO_TC5K1=1 new" timeout 900 bash scripts/gpu_abn.sh bert-large-r16 bert-base-r8 bert-large-r4 2>&1 | head -6
