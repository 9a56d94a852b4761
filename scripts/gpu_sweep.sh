for W in bert-large-r1 bert-large-r2 bert-large-r8 bert-large-r16 bert-large-r32 resnet152-r4 bert-base-r8; do
  timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --secondary none > gpurun_out/sweep_$W.log 2>&1; echo $W rc=$?
done
