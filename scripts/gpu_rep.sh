# repeat the full-size BERT-L r=4 parity test N times (intermittent-failure hunt)
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_rep.log 2>&1
for i in $(seq 1 ${N:-6}); do
  timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "bert-large-4-None" > gpurun_out/rep_$i.log 2>&1; echo "rep $i rc=$?"; grep -E "rel err|passed|failed" gpurun_out/rep_$i.log | head -3
done
