mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_tc5.log 2>&1 || { cat gpurun_out/build_tc5.log; exit 1; }
VARIANTS="${VARS:-new new:ACP_TC5_DBG=7 new:ACP_TC5_DBG=15 new:ACP_TC5_DBG=23 new:ACP_TC5_DBG=31 new:ACP_TC5_DBG=39 new:ACP_TC5_DBG=32}" timeout 900 bash scripts/gpu_abn.sh ${WL:-bert-large-r8} 2>&1 | head -${NL:-7}
