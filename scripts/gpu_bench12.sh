# default bench at N=1 and N=2 (checks the JSON line fields)
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/b1.log 2>&1; echo b1_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/b2.log 2>&1; echo b2_rc=$?
for f in b1 b2; do python - $f <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/{sys.argv[1]}.log").read().strip().splitlines()[-1])
print(sys.argv[1], d["n_gpus"], "ms", round(d["ms_per_step"], 4), "stats", {k: (round(v, 4) if v else v) for k, v in d["step_stats"].items()},
      "nvlink", d["nvlink"], "ssgd", d["ssgd"], "cpu", d["cpu_baseline"], "psgd", (d["powersgd"] or {}).get("acp_speedup"))
PY
done
