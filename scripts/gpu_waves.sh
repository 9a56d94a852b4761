for W in 1 2 4 8; do
  ACP_STREAM_WAVES=$W timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_w$W.log 2>&1; echo W=$W rc=$?
done
