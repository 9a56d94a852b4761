set -x
for D in 0 1; do
  if [ $D = 1 ]; then export ACP_NO_DEFER=1; fi
  timeout 300 python bench.py --workload bert-large-r8 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-powersgd --secondary none > gpurun_out/r8_$D.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/r8_$D.log').read().strip().splitlines()[-1]);pc=d['roofline']['per_class']
print('nodefer=$D', d['ms_per_step'], {k:round(v['ms_per_launch'],4) for k,v in pc.items()})"
done
