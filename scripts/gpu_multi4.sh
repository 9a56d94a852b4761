nvidia-smi -L
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29533 tests/mgpu_check.py > gpurun_out/mgpu4.log 2>&1; echo mgpu4_rc=$?
tail -2 gpurun_out/mgpu4.log
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_n$N.log 2>&1; echo bench$N rc=$?
done
