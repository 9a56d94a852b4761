"""Run-to-run determinism of the whole step on real model shapes: the same
seeded steps run several times through the library must give bit-identical
decoded gradients and state (P, Q, E) -- every reduction in the kernels has a
fixed order, so any difference is a race. This is how the round-2 K1-Q'
race (staged P rows read after the stage release, one warp's column half of
a Q factor off by ~5e-4 once in five runs) was caught
(`scripts/race_probe.py`)."""
import numpy as np
import pytest

from conftest import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA GPU")]


@pytest.mark.parametrize("model,rank,reps", [("bert-base", 2, 4), ("resnet50", 4, 4),
                                             ("bert-base", 8, 3), ("bert-base", 32, 2)])
def test_bitwise_run_to_run(model, rank, reps):
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
    from race_probe import run
    from acp_inputs import gradient_for_shape, ready_order
    shapes = [s for _, s in ready_order(model)]
    steps = 4
    host = [[np.ascontiguousarray(gradient_for_shape(s, seed=11, worker=0, layer=i, step=t))
             for i, s in enumerate(shapes)] for t in range(steps)]
    base = run(shapes, rank, steps, host)
    for _ in range(1, reps):
        o = run(shapes, rank, steps, host)
        for t in range(steps):
            for i in range(len(shapes)):
                assert np.array_equal(o[t][0][i], base[t][0][i]), (t, i, shapes[i], "decoded")
                if o[t][1][i] is not None:
                    for nm, a, b in zip("PQE", o[t][1][i], base[t][1][i]):
                        assert np.array_equal(a, b), (t, i, shapes[i], nm)
