"""World-size-2 host logic on CPU (gloo): the NCCL unique-id broadcast used to
bootstrap the library's communicator, the bench's max-over-ranks timing rule,
and that every rank derives the identical fusion plan (ranks must issue the
same bucket sequence)."""
import os
import sys

import pytest
import torch.multiprocessing as mp

from conftest import ROOT, ensure_built


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2306_08881_b200.acp import broadcast_unique_id
        import bench
        from oracle import fusion_plan
        from acp_inputs import ready_order
        uid = bytes([rank * 7 + i % 251 for i in range(128)]) if rank == 0 else bytes(128)
        got = broadcast_unique_id(uid)
        mx = bench.max_over_ranks(1.5 + rank)
        plan = fusion_plan([s for _, s in ready_order("resnet50")], 4)
        q.put((rank, got, mx, plan["buckets"], plan["slot_off"]))
    finally:
        dist.destroy_process_group()


def test_two_rank_host_logic_gloo():
    ensure_built()  # the binding import needs the built library
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29611
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, id0, mx0, b0, o0), (r1, id1, mx1, b1, o1) = res
    assert id0 == id1 == bytes([i % 251 for i in range(128)])
    assert mx0 == mx1 == 2.5
    assert b0 == b1 and o0 == o1
