set -x
nvidia-smi -L
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29533 tests/mgpu_check.py > gpurun_out/mgpu.log 2>&1; echo mgpu_rc=$?
tail -5 gpurun_out/mgpu.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench2.log 2>&1; echo bench2_rc=$?
tail -c 1500 gpurun_out/bench2.log
