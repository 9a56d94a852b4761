"""Counter-based N(0,1) generator for the random numbers ACP-SGD itself draws.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The method draws random numbers in three places:
  * Q_0 "initialized randomly from standard normal distribution"
    ("i.i.d. standard normal");
  * the rank-deficiency repair of the orthogonaliser (SURVEY.md §8(c) C6,
    SPEC.md S:63 "replace the offending column with a fresh seeded random
    column");
  * the reuse-off ablation (reading C12 in DESIGN.md).

The oracle and the CUDA path each implement THIS SAME counter-based generator
(no shared code): a column of length L for key (seed, tag, layer, step, col)
is, for row i = 0..L-1,

    key = sm64(sm64(sm64(sm64(sm64(seed) ^ tag) ^ layer) ^ step) ^ col)
    a   = sm64(key ^ (2 i)),   b = sm64(key ^ (2 i + 1))
    U1  = ((a >> 11) + 1) * 2^-53        in (0, 1]
    U2  =  (b >> 11)      * 2^-53        in [0, 1)
    z   = sqrt(-2 ln U1) * cos(2 pi U2)  (Box-Muller, float64)

rounded to float32 (factors are stored in fp32), where sm64 is splitmix64:
    x += 0x9E3779B97F4A7C15; x = (x ^ x>>30) * 0xBF58476D1CE4E5B9;
    x = (x ^ x>>27) * 0x94D049BB133111EB; x ^= x>>31      (all mod 2^64)
"""
from __future__ import annotations

import numpy as np

TAG_Q0 = 1
TAG_DEGENERATE = 2
TAG_NO_REUSE = 3

_M = (1 << 64) - 1


def _sm64_int(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M
    return x ^ (x >> 31)


def _sm64_arr(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def column_key(seed: int, tag: int, layer: int, step: int, col: int) -> int:
    k = _sm64_int(int(seed) & _M)
    for v in (tag, layer, step, col):
        k = _sm64_int(k ^ (int(v) & _M))
    return k


def gaussian_column(seed: int, tag: int, layer: int, step: int, col: int,
                    length: int) -> np.ndarray:
    """float64 array holding float32-rounded N(0,1) draws (see module doc)."""
    key = np.uint64(column_key(seed, tag, layer, step, col))
    i = np.arange(length, dtype=np.uint64)
    a = _sm64_arr(key ^ (np.uint64(2) * i))
    b = _sm64_arr(key ^ (np.uint64(2) * i + np.uint64(1)))
    u1 = ((a >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53
    u2 = (b >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    return z.astype(np.float32).astype(np.float64)


def gaussian_factor(seed: int, tag: int, layer: int, step: int, rows: int,
                    r: int) -> np.ndarray:
    """rows x r factor whose column k is gaussian_column(..., col=k)."""
    return np.stack([gaussian_column(seed, tag, layer, step, k, rows) for k in range(r)],
                    axis=1)
