# r <= 4 workloads with the tensor-core path forced (ACP_TC=1) vs default
for W in resnet50-r4 resnet152-r4 bert-large-r4; do
  for TC in 0 1; do
    ACP_TC=$TC timeout 300 python bench.py --workload $W --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-powersgd --secondary none > gpurun_out/tclow_${W}_$TC.log 2>&1
    python - "$W" "$TC" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/tclow_{sys.argv[1]}_{sys.argv[2]}.log").read().strip().splitlines()[-1])
pc = d["roofline"]["per_class"]
print(sys.argv[1], "TC" if sys.argv[2] == "1" else "SIMT", "ms/step %.4f" % d["ms_per_step"], " ".join("%s=%.4f" % (k, v["ms_per_launch"]) for k, v in pc.items()))
PY
  done
done
