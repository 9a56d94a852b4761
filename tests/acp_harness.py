"""Test harness: run the CUDA path (through the C ABI) and the oracle on the
same seeded inputs, and compare per tensor (north_star: relative Frobenius
error <= 1e-4 per layer, fp32)."""
from __future__ import annotations

import numpy as np

from acp_inputs import gradient_for_shape, initial_factor
from oracle import AcpOracle, rel_frobenius

TOL = 1e-4


def make_inputs(shapes, p, steps, seed, recipe="lowrank"):
    return [[[gradient_for_shape(s, seed=seed, worker=w, layer=i, step=t, recipe=recipe)
              for i, s in enumerate(shapes)] for w in range(p)] for t in range(steps)]


def make_q0(shapes, rank, seed):
    q0 = []
    for i, s in enumerate(shapes):
        if len(s) == 1:
            q0.append(None)
            continue
        n, m = s[0], int(np.prod(s[1:]))
        q0.append(initial_factor(m, min(rank, n, m), seed=seed, layer=i))
    return q0


def run_gpu_simulated(shapes, rank, inputs, *, q0=None, seed=0, flags=0, parities=None,
                      bucket_bytes=25 * 2 ** 20, collect_state=True):
    """p simulated workers on one GPU via the split API (acp_compress ->
    element-wise sum of the fused buffers -> acp_decompress)."""
    import torch
    from paper_2306_08881_b200 import AcpContext
    p = len(inputs[0])
    ctxs = [AcpContext(shapes, rank, world_size=p, seed=seed, q0=q0, flags=flags,
                       bucket_bytes=bucket_bytes) for _ in range(p)]
    out = []
    for t, step_in in enumerate(inputs):
        parity = parities[t] if parities else t % 2
        grads = [[torch.from_numpy(np.ascontiguousarray(g)).cuda() for g in step_in[w]]
                 for w in range(p)]
        bufs = [ctxs[w].compress(grads[w], parity) for w in range(p)]
        total = bufs[0].clone()
        for b in bufs[1:]:
            total += b
        for b in bufs:
            b.copy_(total)
        for w in range(p):
            ctxs[w].decompress(grads[w], parity)
        torch.cuda.synchronize()
        rec = {"decoded": [[g.cpu().numpy() for g in grads[w]] for w in range(p)]}
        if collect_state:
            rec["E"] = []
            for w in range(p):
                es = {}
                for i, s in enumerate(shapes):
                    if len(s) > 1:
                        P, Q, E = ctxs[w].get_state(i)
                        es[i] = (P.cpu().numpy(), Q.cpu().numpy(), E.cpu().numpy())
                rec["E"].append(es)
        out.append(rec)
    for c in ctxs:
        c.close()
    return out


def run_oracle(shapes, rank, inputs, *, q0=None, seed=0, ef=True, reuse=True, mean=True,
               parities=None):
    p = len(inputs[0])
    o = AcpOracle(shapes, rank, world_size=p, seed=seed, q0=q0, ef=ef, reuse=reuse, mean=mean)
    out = []
    for t, step_in in enumerate(inputs):
        parity = parities[t] if parities else t % 2
        Eprev = [{i: e.copy() for i, e in o.E[w].items()} for w in range(p)]
        d = o.step(step_in, parity)
        out.append({"decoded": d, "E": [{i: e.copy() for i, e in o.E[w].items()} for w in range(p)],
                    "Eprev": Eprev, "P": dict(o.P), "Q": dict(o.Q)})
    return out


def compare(shapes, gpu, ref, inputs, tol=TOL, check_state=True):
    """Return the worst relative errors; assert all within tol."""
    worst = {"decoded": 0.0, "E": 0.0}
    p = len(inputs[0])
    for t in range(len(ref)):
        for i, s in enumerate(shapes):
            d_ref = ref[t]["decoded"][i]
            for w in range(p):
                e = rel_frobenius(gpu[t]["decoded"][w][i], d_ref)
                if np.linalg.norm(d_ref) == 0:
                    e = float(np.abs(gpu[t]["decoded"][w][i]).max())
                worst["decoded"] = max(worst["decoded"], e)
                assert e <= tol, f"step {t} tensor {i} {s} worker {w}: decoded rel err {e:.3e}"
            if check_state and len(s) > 1 and "E" in gpu[t]:
                for w in range(p):
                    n, m = s[0], int(np.prod(s[1:]))
                    scale = np.linalg.norm(np.float64(inputs[t][w][i]).reshape(n, m) + ref[t]["Eprev"][w][i])
                    E_gpu = gpu[t]["E"][w][i][2]
                    e = rel_frobenius(E_gpu, ref[t]["E"][w][i], scale=scale if scale > 0 else 1.0)
                    worst["E"] = max(worst["E"], e)
                    assert e <= tol, f"step {t} tensor {i} {s} worker {w}: E rel err {e:.3e}"
    return worst
