"""Multi-GPU parity check, launched with torchrun (one process per GPU).

Each rank is one data-parallel worker: it steps its own seeded gradients
through acp_step (per-bucket NCCL all-reduce over NVLink), and compares the
decoded gradients with the oracle run over ALL workers' inputs; decoded
gradients must also be bit-identical across ranks.

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/mgpu_check.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from acp_harness import make_inputs, make_q0, TOL  # noqa: E402
from oracle import AcpOracle, PowerSgdOracle, rel_frobenius  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    from paper_2306_08881_b200 import (AcpContext, nccl_comm_from_group, nccl_comm_destroy,
                                       ACP_POWERSGD)
    comm = nccl_comm_from_group()
    seed = 2306088
    shapes = [(1000,), (64, 3, 7, 7), (2, 1024), (300, 1152), (17,), (512, 4608), (130, 20),
              (1024, 1024), (8, 8)]
    rank_r = 4
    steps = 6
    inputs = make_inputs(shapes, world, steps, seed, "lowrank")
    q0 = make_q0(shapes, rank_r, seed)
    worst = 0.0
    # paper rule, one tensor per bucket, one bucket; the Power-SGD baseline;
    # then the NVLS all-reduce (symmetric memory) with the paper rule and the
    # bucket API
    # ... and the tensor-core path (rank 8: tcgen05 decodes) with NCCL and
    # with the NVLS reduction fused into the tcgen05 decode's prologue
    runs = [(25 * 2 ** 20, 0, False, 4), (0, 0, False, 4), (-1, 0, False, 4),
            (25 * 2 ** 20, ACP_POWERSGD, False, 4), (25 * 2 ** 20, 0, True, 4), (0, 0, True, 4),
            (25 * 2 ** 20, 0, False, 8), (25 * 2 ** 20, 0, True, 8)]
    q0s = {4: q0, 8: make_q0(shapes, 8, seed)}
    for bucket_bytes, flags, nvls, rank_r in runs:
        q0 = q0s[rank_r]
        ctx = AcpContext(shapes, rank_r, world_size=world, nccl_comm=comm, seed=seed, q0=q0,
                         bucket_bytes=bucket_bytes, flags=flags)
        if nvls and not ctx.attach_symmetric():
            if rank == 0:
                print("NVLS multicast unavailable: skipped")
            ctx.close()
            continue
        oc = PowerSgdOracle if flags else AcpOracle
        if rank == 0:
            print(f"run rank={rank_r} bucket_bytes={bucket_bytes} flags={flags} nvls={nvls}", flush=True)
        o = oc(shapes, rank_r, world_size=world, seed=seed, q0=q0)
        for t in range(steps):
            g = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in inputs[t][rank]]
            if bucket_bytes == 0 and not flags:
                # the bucket-granular (WFBP) API, buckets made ready in reverse order
                ctx.step_begin(g, t % 2)
                for b in reversed(range(len(ctx.buckets(t % 2)))):
                    ctx.bucket_ready(b)
                ctx.step_end()
            else:
                ctx.step(g, t % 2)
            ref = o.step(inputs[t], t % 2)
            torch.cuda.synchronize()
            for i, (a, b) in enumerate(zip(g, ref)):
                e = rel_frobenius(a.cpu().numpy(), b)
                worst = max(worst, e)
                assert e <= TOL, f"rank {rank} step {t} tensor {i} {shapes[i]}: rel err {e:.3e}"
                # bit-identical across ranks
                gathered = [torch.empty_like(a) for _ in range(world)]
                dist.all_gather(gathered, a)
                for w in range(world):
                    assert torch.equal(gathered[w], a), f"decoded differs between ranks ({i})"
        ctx.close()
    dist.barrier()
    nccl_comm_destroy(comm)
    if rank == 0:
        print(f"mgpu ok: world={world} worst rel err {worst:.3e}")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
