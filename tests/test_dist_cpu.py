"""World-size-2 host logic on CPU (gloo): the NCCL unique-id broadcast used to
bootstrap the library's communicator, the bench's max-over-ranks timing rule,
and that every rank's LIBRARY derives the identical fusion plan -- ranks must
issue the same bucket sequence -- built by acp_plan_create (the host
half of acp_create) on each rank, gathered over gloo, compared across ranks
and with the oracle's independent plan; and that the cross-rank plan check
(acp.verify_plan_across_ranks) rejects a rank whose layer list differs."""
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
        from paper_2306_08881_b200.acp import broadcast_unique_id, plan_host, verify_plan_across_ranks
        import bench
        from acp_inputs import ready_order
        uid = bytes([rank * 7 + i % 251 for i in range(128)]) if rank == 0 else bytes(128)
        got = broadcast_unique_id(uid)
        mx = bench.max_over_ranks(1.5 + rank)
        shapes = [s for _, s in ready_order("resnet50")]
        plan = plan_host(shapes, 4, world_size=world)
        same = verify_plan_across_ranks(plan)
        # a rank with a different layer list must be caught (not a silent
        # pairing of different buckets)
        bad_shapes = shapes if rank == 0 else shapes[:-1] + [(4096, 64)]
        bad = verify_plan_across_ranks(plan_host(bad_shapes, 4, world_size=world))
        gathered = [None] * world
        dist.all_gather_object(gathered, plan)
        q.put((rank, got, mx, plan, gathered, same, bad))
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
    (r0, id0, mx0, p0, g0, same0, bad0), (r1, id1, mx1, p1, g1, same1, bad1) = res
    assert id0 == id1 == bytes([i % 251 for i in range(128)])
    assert mx0 == mx1 == 2.5
    assert g0 == g1 == [p0, p1] and p0 == p1
    assert same0 and same1 and not bad0 and not bad1
    # the library's plan against the oracle's independent restatement
    from oracle import fusion_plan
    from acp_inputs import ready_order
    want = fusion_plan([s for _, s in ready_order("resnet50")], 4)
    for i, (r, po, qo, eo, bp, bq) in enumerate(p0["tensors"]):
        assert (po, qo, eo) == (want["slot_off"][0][i], want["slot_off"][1][i], want["e_off"][i])
        assert i in want["buckets"][0][bp] and i in want["buckets"][1][bq]
