# Every bench workload on 1 GPU (30 timed steps each, per-kernel classes and the
# on-box Power-SGD comparison); summarised by scripts/summarize_sweep.py.
# usage: bash scripts/gpu_sweep_all.sh TAG
TAG=${1:-sweep}
for W in bert-large-r1 bert-large-r2 bert-large-r4 bert-large-r8 bert-large-r16 bert-large-r32 resnet50-r4 resnet152-r4 bert-base-r8; do
  timeout 600 python bench.py --workload $W --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --secondary none > gpurun_out/${TAG}_$W.log 2>&1; echo $W rc=$?
done
python scripts/summarize_sweep.py $TAG > gpurun_out/${TAG}.md; cat gpurun_out/${TAG}.md
