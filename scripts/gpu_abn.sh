# A/B/n of in-tree builds on one box, interleaved: VARIANTS="base B new" picks
# lib/libacp_<v>.so ("new" = the working-tree lib/libacp.so); "v:VAR=1,VAR2=2" also
# sets environment variables for that variant.
# usage: VARIANTS="base new" bash scripts/gpu_abn.sh [--tests] [workload ...]
if [ "$1" = "--tests" ]; then shift
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/ab_tests.log
fi
for REP in 1 2; do
for W in ${@:-bert-large-r4 resnet50-r4}; do
for VE in ${VARIANTS:-base new}; do
  V=${VE%%:*}; EV=""; [ "$V" != "$VE" ] && EV=${VE#*:}; EV=${EV//,/ }
  if [ $V = new ]; then LIBP=""; else LIBP=$PWD/paper_2306_08881_b200/lib/libacp_$V.so; fi
  env ${LIBP:+ACP_LIB=$LIBP} $EV timeout 300 python bench.py --workload $W --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-powersgd --secondary none > gpurun_out/ab_$W.log 2>&1
  python - "$W" "$VE" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.log").read().strip().splitlines()[-1])
    pc = d["roofline"]["per_class"]
    print("%-14s" % sys.argv[2], sys.argv[1], "ms/step %.4f" % d["ms_per_step"], " ".join("%s=%.4f" % (k, v["ms_per_launch"]) for k, v in pc.items()))
except Exception as e:
    print(sys.argv[2], sys.argv[1], "FAILED", e)
PY
done; done; done
