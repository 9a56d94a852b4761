"""GPU parity of the Power-SGD baseline path (ACP_POWERSGD, SURVEY §8 NEXT-1;
P:180-185, the method ACP-SGD is measured against) vs oracle.PowerSgdOracle.
Same tolerance as the ACP path: relative Frobenius error <= 1e-4 per tensor
per step; E normalised by ||M + E_prev||."""
import numpy as np
import pytest

from conftest import cuda_available
from acp_harness import make_inputs, make_q0, TOL
from oracle import PowerSgdOracle, rel_frobenius

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA GPU")]

SEED = 2306088


def _gpu_split(shapes, rank, inputs, q0, bucket_bytes=25 * 2 ** 20):
    """p simulated workers via the split API: compress(0) -> sum(P) ->
    compress(1) -> sum(Q) -> decompress(1)."""
    import torch
    from paper_2306_08881_b200 import AcpContext, ACP_POWERSGD
    p = len(inputs[0])
    ctxs = [AcpContext(shapes, rank, world_size=p, seed=SEED, q0=q0, flags=ACP_POWERSGD,
                       bucket_bytes=bucket_bytes) for _ in range(p)]
    out = []
    for step_in in inputs:
        grads = [[torch.from_numpy(np.ascontiguousarray(g)).cuda() for g in step_in[w]]
                 for w in range(p)]
        for parity in (0, 1):
            bufs = [ctxs[w].compress(grads[w], parity) for w in range(p)]
            total = bufs[0].clone()
            for b in bufs[1:]:
                total += b
            for b in bufs:
                b.copy_(total)
        for w in range(p):
            ctxs[w].decompress(grads[w], 0)  # no-op for Power-SGD
            ctxs[w].decompress(grads[w], 1)
        torch.cuda.synchronize()
        rec = {"decoded": [[g.cpu().numpy() for g in grads[w]] for w in range(p)], "E": []}
        for w in range(p):
            rec["E"].append({i: ctxs[w].get_state(i)[2].cpu().numpy()
                             for i, s in enumerate(shapes) if len(s) > 1})
        out.append(rec)
    for c in ctxs:
        c.close()
    return out


def _oracle(shapes, rank, inputs, q0):
    p = len(inputs[0])
    o = PowerSgdOracle(shapes, rank, world_size=p, seed=SEED, q0=q0)
    out = []
    for step_in in inputs:
        Eprev = [{i: e.copy() for i, e in o.E[w].items()} for w in range(p)]
        d = o.step(step_in)
        out.append({"decoded": d, "Eprev": Eprev,
                    "E": [{i: e.copy() for i, e in o.E[w].items()} for w in range(p)]})
    return out


def _compare(shapes, gpu, ref, inputs):
    p = len(inputs[0])
    worst = 0.0
    for t in range(len(ref)):
        for i, s in enumerate(shapes):
            d_ref = ref[t]["decoded"][i]
            for w in range(p):
                e = rel_frobenius(gpu[t]["decoded"][w][i], d_ref)
                worst = max(worst, e)
                assert e <= TOL, f"step {t} tensor {i} {s} worker {w}: decoded rel err {e:.3e}"
                if len(s) > 1:
                    n, m = s[0], int(np.prod(s[1:]))
                    scale = np.linalg.norm(np.float64(inputs[t][w][i]).reshape(n, m)
                                           + ref[t]["Eprev"][w][i])
                    e = rel_frobenius(gpu[t]["E"][w][i], ref[t]["E"][w][i],
                                      scale=scale if scale > 0 else 1.0)
                    worst = max(worst, e)
                    assert e <= TOL, f"step {t} tensor {i} {s} worker {w}: E rel err {e:.3e}"
    return worst


RAGGED = [(1000,), (64, 3, 7, 7), (2, 1024), (1, 8), (3, 9000), (64, 64), (256, 64),
          (300, 1152), (17,), (130, 20), (512, 4608), (4, 4)]


@pytest.mark.parametrize("rank", [1, 2, 4, 8, 16, 32])
def test_powersgd_split_api_ragged(rank):
    """r <= 8: the SIMT stream kernels; r = 16 / 32: the register row / column
    kernels (projection-only row kernel, column kernel, row decode)."""
    inputs = make_inputs(RAGGED, 2, 5, SEED, "lowrank")
    q0 = make_q0(RAGGED, rank, SEED)
    print("worst", _compare(RAGGED, _gpu_split(RAGGED, rank, inputs, q0),
                            _oracle(RAGGED, rank, inputs, q0), inputs))


@pytest.mark.parametrize("graphs,rank", [(False, 4), (True, 4), (True, 32)])
def test_powersgd_step_single_worker(graphs, rank):
    """acp_step at world_size 1 (graph replay and eager) vs the oracle with p = 1;
    the parity argument is ignored."""
    import torch
    from paper_2306_08881_b200 import AcpContext, ACP_POWERSGD
    shapes = [(256, 128), (40,), (64, 147), (1024, 1024)]
    inputs = make_inputs(shapes, 1, 6, SEED, "gaussian")
    q0 = make_q0(shapes, rank, SEED)
    ctx = AcpContext(shapes, rank, seed=SEED, q0=q0, flags=ACP_POWERSGD)
    ctx.set_graphs(graphs)
    gpu = []
    for t, step_in in enumerate(inputs):
        g = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in step_in[0]]
        ctx.step(g, t % 2)
        torch.cuda.synchronize()
        gpu.append({"decoded": [[x.cpu().numpy() for x in g]],
                    "E": [{i: ctx.get_state(i)[2].cpu().numpy()
                           for i, s in enumerate(shapes) if len(s) > 1}]})
    ctx.close()
    _compare(shapes, gpu, _oracle(shapes, rank, inputs, q0), inputs)


def test_powersgd_rejects_bad_flags():
    from paper_2306_08881_b200 import AcpContext, AcpError, ACP_POWERSGD, ACP_NO_EF
    with pytest.raises(AcpError):
        AcpContext([(64, 64)], 4, flags=ACP_POWERSGD | ACP_NO_EF)

