"""Full-size parity in bench.py's launch configuration (task: parity at
BASELINE.json's full sizes): the workloads at their real sizes -- BERT-Large
r=4 (bench.py's default line), ResNet-50 r=4, BERT-Base r=8 and BERT-Large
r=32 (tensor-core path), plus BERT-L r=1 and r=8 -- on one GPU through
``AcpContext.step`` with CUDA-graph replay and the default 25 MiB x rate
buckets, i.e. exactly the calls bench.py times, against the fp64 oracle
(oracle/acp_oracle.py, Alg. 2) on the same seeded inputs. FOUR alternating
steps (P, Q, P, Q): the second P-step is the steady state the bench times,
where K1 applies the previous Q-step's deferred residual on the fly (SIMT:
k_stream.cu seg_k1p's `defer` branch; tensor cores: the P_orth Q_loc^T
correction). The oracle finishes these sizes in seconds per step, so every
tensor's decoded gradient is compared in full at every step, and the carried
error-feedback state E of the three largest matrices after every step.
Tolerance: 1e-4 relative Frobenius per tensor (north_star)."""
import numpy as np
import pytest

from conftest import cuda_available
from acp_harness import make_q0, TOL
from acp_inputs import gradient_for_shape, ready_order
from oracle import AcpOracle, rel_frobenius

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA GPU")]

SEED = 2306089


# orth_seg: K2 work-item rows forced through ACP_ORTH_SEG (None = the plan's
# rule). ("bert-large", 1) takes the 1024-row items by default; the forced
# 1024 at r=4 is the case that exposed stale L1 reads of the factor K2
# rewrites in place (profiles/r01_v11_k2_items.md).
STEPS = 4


@pytest.mark.parametrize("model,rank,orth_seg", [("bert-large", 4, None), ("resnet50", 4, None),
                                                 ("bert-base", 8, None), ("bert-large", 32, None),
                                                 ("bert-large", 1, None), ("bert-large", 8, None),
                                                 ("bert-large", 4, "1024")])
def test_full_size_bench_configuration(model, rank, orth_seg, monkeypatch):
    import torch
    if orth_seg is not None:
        monkeypatch.setenv("ACP_ORTH_SEG", orth_seg)  # read by acp_create's plan
    from paper_2306_08881_b200 import AcpContext
    shapes = [s for _, s in ready_order(model)]
    q0 = make_q0(shapes, rank, SEED)
    ctx = AcpContext(shapes, rank, seed=SEED, q0=q0)  # default buckets, world_size 1
    ctx.set_graphs(True)                                # bench.py's timed path
    ref = AcpOracle(shapes, rank, world_size=1, seed=SEED, q0=q0)
    mats = sorted((i for i, s in enumerate(shapes) if len(s) > 1),
                  key=lambda i: -int(np.prod(shapes[i])))[:3]
    worst = [0.0] * STEPS
    for t in range(STEPS):
        e_prev = {i: ref.E[0][i].copy() for i in mats}  # scale of the E comparison
        host = [gradient_for_shape(s, seed=SEED, worker=0, layer=i, step=t)
                for i, s in enumerate(shapes)]
        grads = [torch.from_numpy(np.ascontiguousarray(g)).cuda() for g in host]
        ctx.step(grads, t % 2)
        torch.cuda.synchronize()
        want = ref.step([host], t % 2)
        for i, s in enumerate(shapes):
            got = grads[i].cpu().numpy()
            e = rel_frobenius(got, want[i])
            if np.linalg.norm(want[i]) == 0:
                e = float(np.abs(got).max())
            worst[t] = max(worst[t], e)
            assert e <= TOL, f"{model} r={rank} step {t} tensor {i} {s}: decoded rel err {e:.3e}"
        # carried residual of the three largest matrices (formed by get_state
        # from the implicit state, which stays unchanged), normalised by
        # ||M + E_prev|| as in acp_harness.compare
        for i in mats:
            n, m = shapes[i][0], int(np.prod(shapes[i][1:]))
            _, _, E = ctx.get_state(i)
            scale = np.linalg.norm(np.float64(host[i]).reshape(n, m) + e_prev[i])
            e = rel_frobenius(E.cpu().numpy().reshape(n, m), ref.E[0][i], scale=scale)
            assert e <= TOL, f"{model} r={rank} step {t} tensor {i} {shapes[i]}: E rel err {e:.3e}"
        del grads
    ctx.close()
    print(f"{model} r={rank}: worst decoded rel err per step " + ", ".join(f"{w:.2e}" for w in worst))
