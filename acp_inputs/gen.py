"""Seeded synthetic gradient generators (inputs only; no arithmetic of the method).

Every generator is keyed by (seed, worker, layer, step) through numpy's
SeedSequence, so a given gradient is reproducible and independent of the
order in which others are drawn. Arrays are float32 (the paper trains in
fp32 on RTX 2080 Ti); the oracle promotes them to float64 itself.

Recipes:

* ``lowrank``  - temporally correlated low-rank signal plus full-rank noise,
  mimicking "one can expect that M_t is close to M_{t-1}":
      M_t^w = sum_{k<8} 2^-k u_k v_k^T + 0.1 * N(0,1)/sqrt(m)
  with u_k ~ N(0,1)^n and v_k ~ N(0,1)^m / sqrt(m) fixed per (seed, layer)
  and the noise fresh per (worker, step).
* ``gaussian`` - i.i.d. N(0,1)/sqrt(m), fresh per (worker, step).
* ``uniform``  - i.i.d. U(-1,1)/sqrt(m) (timing inputs; values do not change
  an HBM-bound timing).
"""
from __future__ import annotations

import numpy as np

BASE_SEED = 2306088  # the arXiv id, SURVEY.md §8(d)

_TAG = {"lowrank-signal": 11, "lowrank-noise": 12, "gaussian": 13,
        "uniform": 14, "vector": 15, "q0": 16}


def _rng(seed: int, tag: str, *key: int) -> np.random.Generator:
    return np.random.default_rng([int(seed) & 0xFFFFFFFF, _TAG[tag]] + [int(k) for k in key])


def matrix_gradient(n: int, m: int, *, seed: int, worker: int, layer: int, step: int,
                    recipe: str = "lowrank") -> np.ndarray:
    """One layer's gradient as an (n, m) float32 row-major array."""
    if recipe == "lowrank":
        sig = _rng(seed, "lowrank-signal", layer)
        kmax = 8
        u = sig.standard_normal((n, kmax))
        v = sig.standard_normal((m, kmax)) / np.sqrt(m)
        w = 2.0 ** -np.arange(kmax)
        noise = _rng(seed, "lowrank-noise", worker, layer, step).standard_normal((n, m))
        M = (u * w) @ v.T + 0.1 * noise / np.sqrt(m)
    elif recipe == "gaussian":
        M = _rng(seed, "gaussian", worker, layer, step).standard_normal((n, m)) / np.sqrt(m)
    elif recipe == "uniform":
        M = _rng(seed, "uniform", worker, layer, step).uniform(-1.0, 1.0, (n, m)) / np.sqrt(m)
    else:
        raise ValueError(recipe)
    return np.ascontiguousarray(M, dtype=np.float32)


def vector_gradient(numel: int, *, seed: int, worker: int, layer: int, step: int) -> np.ndarray:
    """A 1-D parameter's gradient (bias / BN / LN), float32."""
    g = _rng(seed, "vector", worker, layer, step).standard_normal(numel)
    return g.astype(np.float32)


def gradient_for_shape(shape, *, seed: int, worker: int, layer: int, step: int,
                       recipe: str = "lowrank") -> np.ndarray:
    """A gradient with the parameter's own shape (k-D or 1-D), float32."""
    shape = tuple(int(d) for d in shape)
    if len(shape) == 1:
        return vector_gradient(shape[0], seed=seed, worker=worker, layer=layer, step=step)
    n = shape[0]
    m = int(np.prod(shape[1:]))
    return matrix_gradient(n, m, seed=seed, worker=worker, layer=layer, step=step,
                           recipe=recipe).reshape(shape)


def initial_factor(m: int, r: int, *, seed: int, layer: int) -> np.ndarray:
    """A shared N(0,1) start factor Q0 (m x r), float32 ("P_0 and Q_0
    are initialized randomly from standard normal distribution"). Tests pass it
    to BOTH sides (oracle argument / library ``q0_host``)."""
    return _rng(seed, "q0", layer).standard_normal((m, r)).astype(np.float32)
