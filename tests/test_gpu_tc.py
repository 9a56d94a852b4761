"""GPU parity of the tensor-core K1 path (k_tc.cu: mma.sync TF32 in 3xTF32
form, double-deferred residual). It is the default for r >= 8;
ACP_TC=1 forces it at lower ranks so every rank class is covered here.
Tolerance as everywhere: relative Frobenius <= 1e-4 per tensor per step."""
import os

import numpy as np
import pytest

from conftest import cuda_available
from acp_harness import make_inputs, make_q0, run_gpu_simulated, run_oracle, compare

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA GPU")]

SEED = 2306088
RAGGED = [(1000,), (64, 3, 7, 7), (2, 1024), (1, 8), (3, 9000), (64, 64), (256, 64), (5, 3, 2),
          (300, 1152), (17,), (130, 20), (512, 4608), (4, 4), (1000, 1024)]


@pytest.fixture
def force_tc(monkeypatch):
    monkeypatch.setenv("ACP_TC", "1")


@pytest.mark.parametrize("rank", [1, 4])
def test_tc_forced_low_rank(force_tc, rank):
    inputs = make_inputs(RAGGED, 2, 6, SEED, "lowrank")
    q0 = make_q0(RAGGED, rank, SEED)
    gpu = run_gpu_simulated(RAGGED, rank, inputs, q0=q0, seed=SEED)
    ref = run_oracle(RAGGED, rank, inputs, q0=q0, seed=SEED)
    print("worst", compare(RAGGED, gpu, ref, inputs))


@pytest.mark.parametrize("parities", [[0, 0, 1, 1, 0, 1], [1, 1, 0, 0, 1]])
def test_tc_irregular_parities(parities):
    """Repeated P- or Q-steps force the host to fold the implicit residual into
    S (tc_materialize_all) before the next projection."""
    shapes = [(96, 80), (80,), (33, 257), (300, 1152)]
    inputs = make_inputs(shapes, 2, len(parities), SEED, "gaussian")
    q0 = make_q0(shapes, 8, SEED)
    gpu = run_gpu_simulated(shapes, 8, inputs, q0=q0, seed=SEED, parities=parities)
    ref = run_oracle(shapes, 8, inputs, q0=q0, seed=SEED, parities=parities)
    compare(shapes, gpu, ref, inputs)


def test_tc_graph_replay_and_determinism():
    import torch
    from paper_2306_08881_b200 import AcpContext
    shapes = [(1024, 1024), (64, 3, 3, 3), (4096,), (512, 4608)]
    outs = []
    for graphs in (True, False, True):
        ctx = AcpContext(shapes, 16, seed=3)
        ctx.set_graphs(graphs)
        gen = torch.Generator(device="cuda").manual_seed(11)
        res = []
        for t in range(4):
            g = [torch.randn(s, device="cuda", generator=gen) for s in shapes]
            ctx.step(g, t % 2)
            res.append([x.clone() for x in g])
        torch.cuda.synchronize()
        outs.append(res)
        ctx.close()
    for a, b in zip(outs[0], outs[1]):
        for x, y in zip(a, b):
            assert torch.equal(x, y)
    for a, b in zip(outs[0], outs[2]):
        for x, y in zip(a, b):
            assert torch.equal(x, y)


# -- kernel selection on the tensor-core path: the tcgen05 decodes (k_tc5.cu,
# default for r >= 8) and tcgen05 K1 P-step (k_tc5k1.cu, default at r = 32)
# forced on / off at every tensor-core rank, so each kernel variant meets the
# oracle on the ragged set (m % 4 != 0 layers, rank clamps, vectors).
@pytest.mark.parametrize("env", [{"ACP_TC5K1": "1"}, {"ACP_TC5K1": "0"}, {"ACP_NO_TC5": "1"}])
@pytest.mark.parametrize("rank", [8, 16, 32])
def test_tc_kernel_variants(monkeypatch, env, rank):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    inputs = make_inputs(RAGGED, 2, 5, SEED, "lowrank")
    q0 = make_q0(RAGGED, rank, SEED)
    gpu = run_gpu_simulated(RAGGED, rank, inputs, q0=q0, seed=SEED)
    ref = run_oracle(RAGGED, rank, inputs, q0=q0, seed=SEED)
    compare(RAGGED, gpu, ref, inputs)


def test_tc5k1_unaligned_gradients_fall_back():
    """The tcgen05 K1 streams M through TMA and needs 16-byte-aligned
    gradients; misaligned views switch the step to the mma.sync kernel (and
    re-capture the graph) with identical results to the oracle."""
    import torch
    from paper_2306_08881_b200 import AcpContext
    from oracle import AcpOracle, rel_frobenius
    shapes = [(300, 1024), (64,), (130, 256)]
    q0 = make_q0(shapes, 32, SEED)
    ctx = AcpContext(shapes, 32, seed=SEED, q0=q0)
    o = AcpOracle(shapes, 32, seed=SEED, q0=q0)
    for t in range(6):
        g = [np.random.default_rng([t, i]).standard_normal(s).astype(np.float32) for i, s in enumerate(shapes)]
        views = []
        for x in g:
            off = 1 if t in (2, 3) else 0      # steps 2-3: 4-byte offset, not 16-byte aligned
            base = torch.empty(x.size + off, device="cuda")
            v = base[off:].view(x.shape)
            v.copy_(torch.from_numpy(x))
            views.append(v)
        ctx.step(views, t % 2)
        ref = o.step([g], t % 2)
        for a, b in zip(views, ref):
            assert rel_frobenius(a.cpu().numpy(), b) < 1e-4
    ctx.close()
