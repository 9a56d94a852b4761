for WV in 1 2 3; do
  for W in resnet50-r4 bert-large-r4; do
  ACP_STREAM_WAVES=$WV timeout 300 python bench.py --workload $W --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-powersgd --secondary none > gpurun_out/wv_$WV.log 2>&1
  python - $WV $W <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/wv_{sys.argv[1]}.log").read().strip().splitlines()[-1])
pc = d["roofline"]["per_class"]
print("waves", sys.argv[1], sys.argv[2], "ms/step %.4f" % d["ms_per_step"], " ".join("%s=%.4f" % (k, v["ms_per_launch"]) for k, v in pc.items()))
PY
  done
done
