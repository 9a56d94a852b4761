"""Plain CPU oracle of ACP-SGD (Alg. 2) and Power-SGD (Alg. 1), float64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Slow and literal on
purpose: every function follows PAPER.md (``P:n`` = line n) step by step, in
the paper's order and notation, with numpy matmul as the only library
primitive. Readings of silent / ambiguous points are SURVEY.md §8(c) C1-C14,
restated in DESIGN.md "Readings".

Conventions
-----------
* Gradients arrive per worker as float32 arrays in the parameter's own shape;
  the oracle promotes them to float64 and computes in float64 throughout
  (reading C11).
* ``parity`` 0 = P-step (the paper's odd t, first step), 1 = Q-step (C1).
* All-reduce = rank-ordered float64 sum ("All-Reduce"; SPEC S:158
  reference reduce). The stored fresh factor is the SUM; the returned
  (decoded) gradient is sum / p unless ``mean=False`` (C2).
* Error feedback uses the LOCAL fresh factor, before aggregation (P:211
  "update the local error ... before aggregation"; Alg. 2 line order
  P:222 before P:223) (C3).
* Orthogonalize = reduced-QR Q factor ("torch.linalg.qr ... reduced QR
  decomposition") computed by modified Gram-Schmidt applied twice, R_kk > 0
  (C5); a column whose residual is <= 1e-6 of its norm (or zero) is replaced
  by a seeded Gaussian column keyed (seed, layer, step, k) (C6).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import rng

DEGENERATE_RTOL = 1e-6          # reading C6
DEFAULT_BUCKET_BYTES = 25 * 2 ** 20   # P:253 "the default buffer size in PyTorch-DDP is 25MB"
MIN_BUCKET_BYTES = 1024          # SPEC S:316 floor, reading C10


# ---------------------------------------------------------------------------
# Shape policy (reading C9) and rank clamp (reading C7)
# ---------------------------------------------------------------------------
def reshape_policy(shape: Sequence[int]) -> Tuple[int, int, bool]:
    """P:260 "The vector-shaped parameters (e.g., biases) requires no
    compression, while other parameters are reshaped into matrices":
    n = dim0, m = prod(dims[1:]); 1-D -> (numel, 1, not compressible)."""
    shape = tuple(int(d) for d in shape)
    if len(shape) == 0 or any(d < 1 for d in shape):
        raise ValueError(f"invalid shape {shape}")
    if len(shape) == 1:
        return shape[0], 1, False
    return shape[0], int(np.prod(shape[1:])), True


def layer_rank(r: int, n: int, m: int) -> int:
    """r_i = min(r, n_i, m_i) (reading C7; "1 <= r <= min(n, m)")."""
    return max(1, min(int(r), int(n), int(m)))


# ---------------------------------------------------------------------------
# Orthogonalize (Alg. 1/2 "Orthogonalize")
# ---------------------------------------------------------------------------
class DegenerateFactor(ValueError):
    pass


def _mgs_pass(A: np.ndarray, fill) -> np.ndarray:
    """One modified Gram-Schmidt sweep, column by column (left to right)."""
    rows, r = A.shape
    Q = np.zeros((rows, r), dtype=np.float64)
    for k in range(r):
        a = A[:, k].astype(np.float64)
        na = math.sqrt(float(a @ a))
        v = a.copy()
        for j in range(k):
            v = v - (Q[:, j] @ v) * Q[:, j]
        nv = math.sqrt(float(v @ v))
        if na == 0.0 or nv <= DEGENERATE_RTOL * na:
            if fill is None:
                raise DegenerateFactor(f"column {k} is (numerically) dependent")
            v = np.asarray(fill(k), dtype=np.float64).copy()
            for j in range(k):
                v = v - (Q[:, j] @ v) * Q[:, j]
            nv = math.sqrt(float(v @ v))
        Q[:, k] = v / nv
    return Q


def orthogonalize(A: np.ndarray, fill=None) -> np.ndarray:
    """Reduced-QR Q factor of a tall rows x r matrix, R_kk > 0 (MGS twice).

    ``fill(k)`` returns the replacement column for a degenerate column k
    (reading C6); without it a degenerate input raises DegenerateFactor.
    """
    A = np.asarray(A, dtype=np.float64)
    if A.ndim != 2 or A.shape[1] > A.shape[0]:
        raise ValueError(f"orthogonalize expects a tall matrix, got {A.shape}")
    if not np.all(np.isfinite(A)):
        raise ValueError("non-finite input to orthogonalize (SPEC S:63)")
    return _mgs_pass(_mgs_pass(A, fill), fill)


def _fill_for(seed: int, layer: int, step: int, rows: int):
    return lambda k: rng.gaussian_column(seed, rng.TAG_DEGENERATE, layer, step, k, rows)


# ---------------------------------------------------------------------------
# Model-level state
# ---------------------------------------------------------------------------
@dataclass
class Layer:
    index: int          # position in READY order (the ABI's tensor index)
    shape: Tuple[int, ...]
    n: int
    m: int
    compressible: bool
    r: int              # r_i (0 for vectors)


def make_layers(shapes_ready: Sequence[Sequence[int]], rank: int) -> List[Layer]:
    out = []
    for i, s in enumerate(shapes_ready):
        n, m, c = reshape_policy(s)
        out.append(Layer(i, tuple(int(d) for d in s), n, m, c, layer_rank(rank, n, m) if c else 0))
    return out


@dataclass
class AcpOracle:
    """p simulated workers of ACP-SGD with EF (Alg. 2).

    ``q0``: optional list (per tensor, None for vectors) of m_i x r_i initial
    factors; when omitted Q_0 comes from the shared counter-based generator
    (oracle/rng.py, tag TAG_Q0, step 0), as the library does with q0_host=NULL.
    """
    shapes_ready: Sequence[Sequence[int]]
    rank: int
    world_size: int = 1
    seed: int = 0
    q0: Optional[List[Optional[np.ndarray]]] = None
    ef: bool = True
    reuse: bool = True
    mean: bool = True
    layers: List[Layer] = field(init=False)
    P: Dict[int, np.ndarray] = field(init=False)
    Q: Dict[int, np.ndarray] = field(init=False)
    E: List[Dict[int, np.ndarray]] = field(init=False)
    step_count: int = field(init=False, default=0)

    def __post_init__(self):
        self.layers = make_layers(self.shapes_ready, self.rank)
        self.P, self.Q = {}, {}
        self.E = [dict() for _ in range(self.world_size)]
        for L in self.layers:
            if not L.compressible:
                continue
            if self.q0 is not None and self.q0[L.index] is not None:
                q0 = np.asarray(self.q0[L.index], dtype=np.float32).astype(np.float64)
                assert q0.shape == (L.m, L.r), (q0.shape, (L.m, L.r))
            else:
                q0 = rng.gaussian_factor(self.seed, rng.TAG_Q0, L.index, 0, L.m, L.r)
            self.Q[L.index] = q0
            # P_0 is initialised in the paper but never read by Alg. 2
            # (reading C4); keep zeros so the state is fully defined.
            self.P[L.index] = np.zeros((L.n, L.r))
            for w in range(self.world_size):
                self.E[w][L.index] = np.zeros((L.n, L.m))      # E_0 = 0

    # -- Alg. 2, one layer ------------------------------------------------
    def _reused_factor(self, L: Layer, which: str) -> np.ndarray:
        rows = L.m if which == "Q" else L.n
        if self.reuse:
            return self.Q[L.index] if which == "Q" else self.P[L.index]
        # reuse-off ablation (reading C12): a fresh shared factor
        return rng.gaussian_factor(self.seed, rng.TAG_NO_REUSE, L.index, self.step_count,
                                   rows, L.r)

    def _step_layer(self, L: Layer, Ms: List[np.ndarray], parity: int) -> np.ndarray:
        p = self.world_size
        fill_rows = L.m if parity == 0 else L.n
        fill = _fill_for(self.seed, L.index, self.step_count, fill_rows)
        fresh = []
        if parity == 0:                                   # t odd
            Qt = orthogonalize(self._reused_factor(L, "Q"), fill)
            for w in range(p):
                Mp = Ms[w] + (self.E[w][L.index] if self.ef else 0.0)
                Pw = Mp @ Qt
                if self.ef:
                    self.E[w][L.index] = Mp - Pw @ Qt.T
                fresh.append(Pw)
            Pt = reference_reduce(fresh)
            decoded = Pt @ Qt.T
            self.P[L.index], self.Q[L.index] = Pt, Qt
        else:                                             # t even
            Pt = orthogonalize(self._reused_factor(L, "P"), fill)
            for w in range(p):
                Mp = Ms[w] + (self.E[w][L.index] if self.ef else 0.0)
                Qw = Mp.T @ Pt
                if self.ef:
                    self.E[w][L.index] = Mp - Pt @ Qw.T
                fresh.append(Qw)
            Qt = reference_reduce(fresh)
            decoded = Pt @ Qt.T
            self.P[L.index], self.Q[L.index] = Pt, Qt
        return decoded / p if self.mean else decoded

    def step(self, grads: Sequence[Sequence[np.ndarray]], parity: int) -> List[np.ndarray]:
        """grads[w][i]: worker w's gradient of tensor i (ready order, param
        shape, float32). Returns the decoded gradient of every tensor (float64,
        param shape), identical on every worker."""
        if parity not in (0, 1):
            raise ValueError("parity must be 0 (P-step) or 1 (Q-step)")
        if len(grads) != self.world_size:
            raise ValueError("one gradient list per worker")
        out = []
        for L in self.layers:
            Ms = [np.asarray(grads[w][L.index], dtype=np.float64).reshape(L.n, L.m)
                  for w in range(self.world_size)]
            if L.compressible:
                d = self._step_layer(L, Ms, parity)
            else:
                # vectors ride uncompressed in the same fused buffer (
                # reading C8) and are simply all-reduced
                d = reference_reduce(Ms)
                d = d / self.world_size if self.mean else d
            out.append(d.reshape(L.shape))
        self.step_count += 1
        return out


def reference_reduce(xs: Sequence[np.ndarray]) -> np.ndarray:
    """All-Reduce(sum) as a rank-ordered float64 sum."""
    acc = np.array(xs[0], dtype=np.float64, copy=True)
    for x in xs[1:]:
        acc = acc + np.asarray(x, dtype=np.float64)
    return acc


# ---------------------------------------------------------------------------
# Power-SGD (Alg. 1) with error feedback (reading C13)
# ---------------------------------------------------------------------------
@dataclass
class PowerSgdOracle:
    shapes_ready: Sequence[Sequence[int]]
    rank: int
    world_size: int = 1
    seed: int = 0
    q0: Optional[List[Optional[np.ndarray]]] = None
    ef: bool = True
    mean: bool = True
    layers: List[Layer] = field(init=False)
    Q: Dict[int, np.ndarray] = field(init=False)
    E: List[Dict[int, np.ndarray]] = field(init=False)
    step_count: int = field(init=False, default=0)

    def __post_init__(self):
        self.layers = make_layers(self.shapes_ready, self.rank)
        self.Q = {}
        self.E = [dict() for _ in range(self.world_size)]
        for L in self.layers:
            if not L.compressible:
                continue
            if self.q0 is not None and self.q0[L.index] is not None:
                self.Q[L.index] = np.asarray(self.q0[L.index], np.float32).astype(np.float64)
            else:
                self.Q[L.index] = rng.gaussian_factor(self.seed, rng.TAG_Q0, L.index, 0, L.m, L.r)
            for w in range(self.world_size):
                self.E[w][L.index] = np.zeros((L.n, L.m))

    def step(self, grads, parity_unused: int = 0) -> List[np.ndarray]:
        p = self.world_size
        out = []
        for L in self.layers:
            Ms = [np.asarray(grads[w][L.index], dtype=np.float64).reshape(L.n, L.m)
                  for w in range(p)]
            if not L.compressible:
                d = reference_reduce(Ms)
                out.append((d / p if self.mean else d).reshape(L.shape))
                continue
            Mp = [Ms[w] + (self.E[w][L.index] if self.ef else 0.0) for w in range(p)]
            Pt = reference_reduce([Mp[w] @ self.Q[L.index] for w in range(p)])
            Pt = orthogonalize(Pt, _fill_for(self.seed, L.index, self.step_count, L.n))
            Qw = [Mp[w].T @ Pt for w in range(p)]
            Qt = reference_reduce(Qw)
            if self.ef:
                for w in range(p):
                    self.E[w][L.index] = Mp[w] - Pt @ Qw[w].T
            self.Q[L.index] = Qt
            d = Pt @ Qt.T
            out.append((d / p if self.mean else d).reshape(L.shape))
        self.step_count += 1
        return out


# ---------------------------------------------------------------------------
# Tensor-fusion plan (reading C10) and fused-buffer layout
# ---------------------------------------------------------------------------
def payload_elems(L: Layer, parity: int) -> int:
    """Elements tensor L contributes to the parity's fused buffer: the fresh
    factor (n_i r_i on P-steps, m_i r_i on Q-steps) or the whole vector."""
    if not L.compressible:
        return L.n
    return L.n * L.r if parity == 0 else L.m * L.r


def compression_rates(layers: Sequence[Layer]) -> Tuple[float, float]:
    """P:257 "the compression rates of ACP-SGD ... for P and Q", counting the
    uncompressed vectors in the buffers."""
    N = sum(L.n * L.m for L in layers)
    fp = sum(payload_elems(L, 0) for L in layers)
    fq = sum(payload_elems(L, 1) for L in layers)
    return fp / N, fq / N


def buffer_cap_bytes(default_bytes: int, rate: float) -> int:
    """P:257 "configure the compressed buffer size by scaling the default
    buffer size with the compression rate"; ceil, 1 KB floor (C10)."""
    if default_bytes <= 0:
        return default_bytes
    return max(MIN_BUCKET_BYTES, int(math.ceil(default_bytes * rate)))


def plan_buckets(sizes_bytes: Sequence[int], cap: int) -> List[List[int]]:
    """Greedy fill in ready order; seal once total >= cap ("select the
    available tensors to fit in the buffer"). cap == 0: one
    tensor per bucket; cap < 0: a single bucket."""
    if cap < 0:
        return [list(range(len(sizes_bytes)))]
    buckets, cur, tot = [], [], 0
    for i, s in enumerate(sizes_bytes):
        cur.append(i)
        tot += s
        if tot >= cap:
            buckets.append(cur)
            cur, tot = [], 0
    if cur:
        buckets.append(cur)
    return buckets


def _round4(x: int) -> int:
    return (x + 3) // 4 * 4


def fusion_plan(shapes_ready: Sequence[Sequence[int]], rank: int,
                default_bucket_bytes: int = DEFAULT_BUCKET_BYTES) -> dict:
    """Independent restatement of the library's plan (include/acp.h
    "Layout"): per-tensor r_i, 16-byte-aligned slot offsets (floats) in the
    P- and Q-buffers (ready order, each slot padded to a multiple of 4
    floats), E offsets (compressible tensors only, padded the same way), and
    the greedy buckets per parity."""
    layers = make_layers(shapes_ready, rank)
    rate_p, rate_q = compression_rates(layers)
    plan = {"layers": layers, "rate": (rate_p, rate_q), "cap": [], "buckets": [],
            "slot_off": [], "e_off": []}
    e = 0
    for L in layers:
        plan["e_off"].append(e if L.compressible else -1)
        if L.compressible:
            e += _round4(L.n * L.m)
    plan["e_elems"] = e
    for parity, rate in ((0, rate_p), (1, rate_q)):
        cap = buffer_cap_bytes(default_bucket_bytes, rate)
        sizes = [4 * payload_elems(L, parity) for L in layers]
        plan["cap"].append(cap)
        plan["buckets"].append(plan_buckets(sizes, cap))
        offs, o = [], 0
        for L in layers:
            offs.append(o)
            o += _round4(payload_elems(L, parity))
        plan["slot_off"].append(offs)
        plan.setdefault("arena_elems", []).append(o)
    return plan


# ---------------------------------------------------------------------------
# Metrics
# ---------------------------------------------------------------------------
def rel_frobenius(x: np.ndarray, ref: np.ndarray, scale: Optional[float] = None) -> float:
    """||x - ref||_F / scale (scale defaults to ||ref||_F; north_star 1e-4)."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    d = float(np.linalg.norm((x - ref).ravel()))
    s = float(np.linalg.norm(ref.ravel())) if scale is None else float(scale)
    return d / s if s > 0 else d
