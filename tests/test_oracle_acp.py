"""Pins for the ACP-SGD oracle (Alg. 2).

Each test checks the oracle against something it does not compute itself:
closed forms (Eckart-Young, full rank = S-SGD), invariants that a plausible
mistake breaks (residual orthogonal to the reused factor fails if E used the
aggregated factor; linearity fails for a transposed operand), SPEC examples,
and a brute-force pure-Python restatement on tiny shapes that orthogonalises
with Householder QR instead of Gram-Schmidt.
"""
import math

import numpy as np
import pytest

from conftest import golden
from oracle import AcpOracle, PowerSgdOracle, rel_frobenius, rng, payload_elems, make_layers


def _grads(shapes, p, step, seed=1, scale=1.0):
    rs = np.random.default_rng([seed, step])
    return [[(scale * rs.standard_normal(s)).astype(np.float32) for s in shapes]
            for _ in range(p)]


def _hh_orth(A):
    Q, R = np.linalg.qr(A)
    s = np.sign(np.diag(R))
    s[s == 0] = 1
    return Q * s


# -- closed forms -------------------------------------------------------------
@pytest.mark.parametrize("p", [1, 2, 3])
def test_full_rank_square_is_ssgd(p):
    """n = m = r: every projection is onto the whole space, so ACP-SGD reduces
    to S-SGD: decoded = mean of the workers' gradients and E stays 0."""
    shapes = [(6, 6), (6,)]
    o = AcpOracle(shapes, rank=6, world_size=p, seed=3)
    for s in range(6):
        g = _grads(shapes, p, s)
        d = o.step(g, s % 2)
        mean = sum(np.float64(g[w][0]) for w in range(p)) / p
        np.testing.assert_allclose(d[0], mean, atol=1e-12)
        np.testing.assert_allclose(d[1], sum(np.float64(g[w][1]) for w in range(p)) / p, atol=1e-15)
        for w in range(p):
            assert np.abs(o.E[w][0]).max() < 1e-12


def test_full_rank_only_on_square_side():
    """r = m < n: P-steps are exact (Q Q^T = I_m), Q-steps are not
    (P P^T != I_n). Reading of north_star's 'full-rank r=min(n,m)'."""
    shapes = [(12, 4)]
    o = AcpOracle(shapes, rank=4, world_size=1, seed=2)
    g0 = _grads(shapes, 1, 0)
    d0 = o.step(g0, 0)
    np.testing.assert_allclose(d0[0], g0[0][0], atol=1e-12)
    assert np.abs(o.E[0][0]).max() < 1e-12
    g1 = _grads(shapes, 1, 1)
    d1 = o.step(g1, 1)
    assert rel_frobenius(d1[0], g1[0][0]) > 0.1
    # and the mirror case: r = n < m, Q-step exact
    o2 = AcpOracle([(4, 12)], rank=4, world_size=1, seed=2)
    o2.step(_grads([(4, 12)], 1, 0), 0)
    g = _grads([(4, 12)], 1, 1)
    E_prev = o2.E[0][0].copy()
    d = o2.step(g, 1)
    np.testing.assert_allclose(d[0], g[0][0] + E_prev, atol=1e-12)


@pytest.mark.parametrize("embed", [False, True])
def test_eckart_young_rank1_ef_off(embed):
    """fixed M = diag(3,2,1), r = 1, EF off, query reuse: the
    alternating power iteration converges to the best rank-1 approximation,
    ||M - decoded||_F -> sqrt(2^2+1^2) = sqrt(5), monotonically."""
    g = golden("spec_examples.json")
    M = np.diag(np.array(g["rank1_diag"], dtype=np.float32))
    if embed:
        big = np.zeros((256, 128), np.float32)
        big[:3, :3] = M
        rs = np.random.default_rng(0)
        Ul, _ = np.linalg.qr(rs.standard_normal((256, 256)))
        Vr, _ = np.linalg.qr(rs.standard_normal((128, 128)))
        M = (Ul @ big @ Vr.T).astype(np.float32)
    o = AcpOracle([M.shape], rank=1, world_size=1, seed=11, ef=False)
    errs = []
    for s in range(20):
        d = o.step([[M]], s % 2)
        errs.append(float(np.linalg.norm(np.float64(M) - d[0])))
    assert abs(errs[-1] - g["rank1_limit"]) < 1e-3
    assert all(b <= a + 1e-6 for a, b in zip(errs, errs[1:]))


# -- invariants ---------------------------------------------------------------
@pytest.mark.parametrize("p", [1, 2, 4])
def test_conservation_and_local_residual(p):
    """M + E_prev = M_hat_loc + E_new, with M_hat_loc of rank r built from the
    LOCAL fresh factor: the new residual is orthogonal to the
    reused (orthonormal) factor: E_new Q = 0 on P-steps, P^T E_new = 0 on
    Q-steps. Using the aggregated factor instead breaks this for p > 1."""
    shapes = [(20, 9)]
    r = 3
    o = AcpOracle(shapes, rank=r, world_size=p, seed=5)
    for s in range(6):
        Eprev = [o.E[w][0].copy() for w in range(p)]
        g = _grads(shapes, p, s)
        o.step(g, s % 2)
        for w in range(p):
            Mp = np.float64(g[w][0]) + Eprev[w]
            Mhat = Mp - o.E[w][0]
            assert np.linalg.matrix_rank(Mhat, tol=1e-9) <= r
            if s % 2 == 0:
                assert np.abs(o.E[w][0] @ o.Q[0]).max() < 1e-12
                np.testing.assert_allclose(Mhat, Mp @ o.Q[0] @ o.Q[0].T, atol=1e-12)
            else:
                assert np.abs(o.P[0].T @ o.E[w][0]).max() < 1e-12
                np.testing.assert_allclose(Mhat, o.P[0] @ o.P[0].T @ Mp, atol=1e-12)


@pytest.mark.parametrize("p", [1, 3])
def test_ef_telescoping(p):
    """SPEC S:255 / acceptance #5: sum_w E_T^w = sum_{s,w} M_s^w - p sum_s decoded_s
    (p = 1: E_T = sum M - sum decoded)."""
    shapes = [(15, 10), (10,)]
    o = AcpOracle(shapes, rank=2, world_size=p, seed=8)
    sumM = np.zeros((15, 10))
    sumD = np.zeros((15, 10))
    for s in range(9):
        g = _grads(shapes, p, s)
        d = o.step(g, s % 2)
        sumM += sum(np.float64(g[w][0]) for w in range(p))
        sumD += d[0]
    sumE = sum(o.E[w][0] for w in range(p))
    np.testing.assert_allclose(sumE, sumM - p * sumD, atol=1e-10)


def test_linearity_of_aggregation():
    """P:132 additivity / north_star: sum_w (M'_w Q) = (sum_w M'_w) Q for a
    shared Q, so the P-step decoded gradient equals (1/p)(sum_w M'_w) Q Q^T
    with Q = orth(previous aggregated Q) -- computed here with Householder."""
    shapes = [(18, 11)]
    p, r = 3, 4
    o = AcpOracle(shapes, rank=r, world_size=p, seed=21)
    for s in range(5):
        Eprev = [o.E[w][0].copy() for w in range(p)]
        Qprev, Pprev = o.Q[0].copy(), o.P[0].copy()
        g = _grads(shapes, p, s)
        d = o.step(g, s % 2)
        S = sum(np.float64(g[w][0]) + Eprev[w] for w in range(p))
        if s % 2 == 0:
            Qo = _hh_orth(Qprev)
            np.testing.assert_allclose(d[0], S @ Qo @ Qo.T / p, atol=1e-11)
        else:
            Po = _hh_orth(Pprev)
            np.testing.assert_allclose(d[0], Po @ Po.T @ S / p, atol=1e-11)


def test_identical_workers_equal_single_worker():
    """p workers holding identical inputs follow the
    single-worker trajectory."""
    shapes = [(16, 12), (7,), (5, 3, 2)]
    o1 = AcpOracle(shapes, rank=3, world_size=1, seed=4)
    o3 = AcpOracle(shapes, rank=3, world_size=3, seed=4)
    for s in range(7):
        g = _grads(shapes, 1, s)
        d1 = o1.step(g, s % 2)
        d3 = o3.step([g[0]] * 3, s % 2)
        for a, b in zip(d1, d3):
            np.testing.assert_allclose(a, b, atol=1e-12)


def test_first_step_is_p_step_and_halving_law():
    """Alg. 2 t=1 (odd) computes P: payload n*r. The halving law
    (SPEC S:256): ACP sends n r + m r per two steps, Power-SGD 2(n+m)r."""
    g = golden("spec_examples.json")["halving"]
    L = make_layers([(g["n"], g["m"])], g["r"])[0]
    assert payload_elems(L, 0) + payload_elems(L, 1) == g["acp_two_steps"]
    assert 2 * (payload_elems(L, 0) + payload_elems(L, 1)) == g["powersgd_two_steps"]
    o = AcpOracle([(30, 8)], rank=2, world_size=1, seed=1)
    q_before = o.Q[0].copy()
    o.step(_grads([(30, 8)], 1, 0), 0)
    # P-step: the stored Q is orth(Q_0), and P holds the fresh n x r factor
    np.testing.assert_allclose(o.Q[0], _hh_orth(q_before), atol=1e-12)
    assert o.P[0].shape == (30, 2)


def test_zero_gradient_and_degenerate_repair():
    """An all-zero gradient at step 1 makes P = 0; the next Q-step must
    orthogonalise a zero factor: columns are replaced by the seeded Gaussian
    columns (reading C6) and the step stays finite."""
    o = AcpOracle([(10, 6)], rank=2, world_size=1, seed=13)
    z = [[np.zeros((10, 6), np.float32)]]
    d0 = o.step(z, 0)
    assert np.all(d0[0] == 0)
    d1 = o.step(z, 1)
    assert np.all(d1[0] == 0)
    Z = np.stack([rng.gaussian_column(13, rng.TAG_DEGENERATE, 0, 1, k, 10) for k in range(2)], 1)
    np.testing.assert_allclose(o.P[0], _hh_orth(Z), atol=1e-12)


def test_default_q0_comes_from_counter_generator():
    o = AcpOracle([(9, 5)], rank=2, world_size=1, seed=77)
    Z = np.stack([rng.gaussian_column(77, rng.TAG_Q0, 0, 0, k, 5) for k in range(2)], 1)
    np.testing.assert_array_equal(o.Q[0], Z)


def test_no_reuse_uses_fresh_factor():
    """Reuse-off ablation (reading C12): orthogonalise a fresh seeded
    factor each step instead of the previous aggregated one."""
    shapes = [(14, 9)]
    o = AcpOracle(shapes, rank=2, world_size=1, seed=6, reuse=False)
    for s in range(3):
        Eprev = o.E[0][0].copy()
        g = _grads(shapes, 1, s)
        d = o.step(g, s % 2)
        rows = 9 if s % 2 == 0 else 14
        F = _hh_orth(rng.gaussian_factor(6, rng.TAG_NO_REUSE, 0, s, rows, 2))
        Mp = np.float64(g[0][0]) + Eprev
        ref = Mp @ F @ F.T if s % 2 == 0 else F @ F.T @ Mp
        np.testing.assert_allclose(d[0], ref, atol=1e-11)


# -- brute force on tiny shapes ------------------------------------------------
def _bf_matmul(A, B):
    n, k = len(A), len(A[0])
    m = len(B[0])
    return [[sum(A[i][t] * B[t][j] for t in range(k)) for j in range(m)] for i in range(n)]


def _bf_T(A):
    return [list(r) for r in zip(*A)]


def _bf_orth(A):
    Q = _hh_orth(np.array(A, dtype=np.float64))
    return Q.tolist()


def _bf_acp(Ms_per_step, p, r, Q0):
    """Alg. 2 with EF transcribed with Python lists; all-reduce = sum; returns
    decoded (sum / p) and final E per worker."""
    n, m = len(Ms_per_step[0][0]), len(Ms_per_step[0][0][0])
    E = [[[0.0] * m for _ in range(n)] for _ in range(p)]
    P, Q = None, [row[:] for row in Q0]
    outs = []
    for t, Ms in enumerate(Ms_per_step, start=1):
        Mp = [[[Ms[w][i][j] + E[w][i][j] for j in range(m)] for i in range(n)] for w in range(p)]
        if t % 2 == 1:
            Q = _bf_orth(Q)
            fresh = [_bf_matmul(Mp[w], Q) for w in range(p)]
            for w in range(p):
                rec = _bf_matmul(fresh[w], _bf_T(Q))
                E[w] = [[Mp[w][i][j] - rec[i][j] for j in range(m)] for i in range(n)]
            P = [[sum(fresh[w][i][k] for w in range(p)) for k in range(r)] for i in range(n)]
        else:
            P = _bf_orth(P)
            fresh = [_bf_matmul(_bf_T(Mp[w]), P) for w in range(p)]
            for w in range(p):
                rec = _bf_matmul(P, _bf_T(fresh[w]))
                E[w] = [[Mp[w][i][j] - rec[i][j] for j in range(m)] for i in range(n)]
            Q = [[sum(fresh[w][j][k] for w in range(p)) for k in range(r)] for j in range(m)]
        dec = _bf_matmul(P, _bf_T(Q))
        outs.append([[x / p for x in row] for row in dec])
    return outs, E


@pytest.mark.parametrize("n,m,r,p", [(4, 3, 2, 2), (3, 5, 1, 1), (5, 4, 3, 3)])
def test_brute_force_tiny(n, m, r, p):
    rs = np.random.default_rng(n * 31 + m * 7 + r)
    steps = 5
    Ms = [[rs.standard_normal((n, m)).astype(np.float32) for _ in range(p)] for _ in range(steps)]
    Q0 = rs.standard_normal((m, r)).astype(np.float32)
    bf_out, bf_E = _bf_acp([[M.astype(np.float64).tolist() for M in step] for step in Ms], p, r,
                           Q0.astype(np.float64).tolist())
    o = AcpOracle([(n, m)], rank=r, world_size=p, q0=[Q0])
    for s in range(steps):
        d = o.step([[Ms[s][w]] for w in range(p)], s % 2)
        np.testing.assert_allclose(d[0], np.array(bf_out[s]), atol=1e-11)
    for w in range(p):
        np.testing.assert_allclose(o.E[w][0], np.array(bf_E[w]), atol=1e-11)


# -- Power-SGD (Alg. 1) --------------------------------------------------------
def test_powersgd_rank1_monotone_to_sqrt5():
    """Power-SGD on a fixed diag(3,2,1), r=1, EF off:
    monotone nonincreasing error converging to sqrt(5)."""
    M = np.diag([3.0, 2.0, 1.0]).astype(np.float32)
    o = PowerSgdOracle([M.shape], rank=1, world_size=1, seed=2, ef=False)
    errs = [float(np.linalg.norm(np.float64(M) - o.step([[M]])[0])) for _ in range(20)]
    assert abs(errs[-1] - math.sqrt(5)) < 1e-3
    assert all(b <= a + 1e-6 for a, b in zip(errs, errs[1:]))


def test_powersgd_full_rank_exact_and_linear():
    """r = m: Power-SGD's decoded gradient is the mean of the workers' M after
    one step (P P^T projects onto the range of M Q; SPEC powersgd example)."""
    shapes = [(9, 4)]
    o = PowerSgdOracle(shapes, rank=4, world_size=2, seed=3)
    g = _grads(shapes, 2, 0)
    d = o.step(g)
    np.testing.assert_allclose(d[0], (np.float64(g[0][0]) + g[1][0]) / 2, atol=1e-11)


def test_powersgd_identical_workers():
    shapes = [(12, 7)]
    a = PowerSgdOracle(shapes, rank=2, world_size=1, seed=4)
    b = PowerSgdOracle(shapes, rank=2, world_size=2, seed=4)
    for s in range(4):
        g = _grads(shapes, 1, s)
        np.testing.assert_allclose(a.step(g)[0], b.step([g[0], g[0]])[0], atol=1e-12)


# -- Power-SGD error feedback (reading C13, Alg. 1 + P:211) ----------------------
# Alg. 1 prints no error-feedback line; C13 reads it as Alg. 2's:
# E_w = M'_w - P_hat Q_w^T with the orthogonalised aggregated P_hat and the
# worker's LOCAL Q_w = M'_w^T P_hat. The pins below are properties of that
# formula that the alternatives break: E from the aggregated Q (Alg. 2's
# "before aggregation" violated), SPEC's E = M' - decoded, a dropped
# E in M', a sign error.
def _psgd_run(shapes, p, steps, seed=7, ef=True):
    o = PowerSgdOracle(shapes, rank=3, world_size=p, seed=seed, ef=ef)
    for s in range(steps):
        g = _grads(shapes, p, s, seed=seed)
        Mp = [{i: np.float64(g[w][i]).reshape(o.E[w][i].shape) + o.E[w][i] for i in o.E[w]}
              for w in range(p)]
        d = o.step(g)
        yield o, g, Mp, d


def test_powersgd_ef_residual_orthogonal_to_decoded_range():
    """P_hat^T E_w = P_hat^T M'_w - Q_w^T = 0 for the LOCAL Q_w, so every
    worker's residual is orthogonal to the range of the decoded gradient
    (decoded^T E_w = 0). Fails for E from the aggregated Q and for SPEC's
    E = M' - decoded, whenever the workers' inputs differ."""
    shapes = [(20, 9)]
    for o, g, Mp, d in _psgd_run(shapes, 3, 4):
        D = d[0]
        for w in range(3):
            E = o.E[w][0]
            assert np.abs(D.T @ E).max() <= 1e-12 * np.linalg.norm(D) * np.linalg.norm(Mp[w][0])
            assert np.linalg.norm(E) > 1e-3  # not trivially zero (r < rank of M')
    # the alternatives violate it
    o = PowerSgdOracle(shapes, rank=3, world_size=3, seed=7)
    g = _grads(shapes, 3, 0, seed=7)
    d = o.step(g)[0]
    alt = np.float64(g[1][0]) - d                  # SPEC's E = M' - decoded (p > 1)
    assert np.abs(d.T @ alt).max() > 1e-3 * np.linalg.norm(d) * np.linalg.norm(alt)


def test_powersgd_ef_sum_identity_and_conservation():
    """Sum over workers: sum_w E_w = sum_w M'_w - p * decoded (because
    sum_w P_hat Q_w^T = P_hat Q^T = p * decoded). E from the aggregated Q
    would give sum_w M'_w - p^2 * decoded instead."""
    p = 3
    for o, g, Mp, d in _psgd_run([(16, 12), (12,)], p, 4):
        lhs = sum(o.E[w][0] for w in range(p))
        rhs = sum(Mp[w][0] for w in range(p)) - p * d[0]
        assert np.abs(lhs - rhs).max() <= 1e-12 * max(1.0, np.abs(rhs).max())
        assert np.abs(d[0]).max() > 1e-3


def test_powersgd_ef_telescoping_single_worker():
    """p = 1: E_T = sum_s M_s - sum_s decoded_s -- the
    compression error is carried, never lost; a dropped E in M' or a sign
    error breaks it after the second step."""
    shapes = [(14, 10)]
    acc_m = np.zeros((14, 10))
    acc_d = np.zeros((14, 10))
    for o, g, Mp, d in _psgd_run(shapes, 1, 6):
        acc_m += np.float64(g[0][0])
        acc_d += d[0]
        np.testing.assert_allclose(o.E[0][0], acc_m - acc_d, atol=1e-11)


def test_powersgd_ef_feeds_next_step():
    """M' = M + E: an EF-off oracle fed M + E_prev by hand follows the
    EF-on trajectory exactly (same Q state, same decoded gradients)."""
    shapes = [(18, 11)]
    p = 2
    a = PowerSgdOracle(shapes, rank=2, world_size=p, seed=9)
    b = PowerSgdOracle(shapes, rank=2, world_size=p, seed=9, ef=False)
    for s in range(5):
        g = _grads(shapes, p, s, seed=9)
        fed = [[(np.float64(g[w][0]) + a.E[w][0])] for w in range(p)]
        da = a.step(g)[0]
        db = b.step(fed)[0]
        np.testing.assert_allclose(da, db, atol=1e-12)
