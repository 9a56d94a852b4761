# Multi-GPU evidence on one N-GPU box: parity (tests/mgpu_check.py), then
# NCCL vs NVLS ms/step for BERT-L r=4 and ResNet-50 r=4 at N=2 (and N=4 when
# the box has 4 GPUs). usage: bash scripts/gpu_multi_v8.sh N
N=${1:-2}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29533 tests/mgpu_check.py > gpurun_out/mgpu_v8_$N.log 2>&1; echo mgpu_rc=$?
tail -2 gpurun_out/mgpu_v8_$N.log
for M in $(seq 2 $N); do
  [ $M = 2 ] || [ $M = 4 ] || continue
  bash scripts/gpu_nvls.sh $M
done
