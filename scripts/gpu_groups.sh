for G in 1 2 4 8 16; do
  ACP_COMPUTE_GROUPS=$G timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 2954$G bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --secondary resnet50-r4 > gpurun_out/bench2_g$G.log 2>&1; echo G=$G rc=$?
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29560 bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --bucket-bytes -1 > gpurun_out/bench2_single.log 2>&1; echo single rc=$?
