"""Pins for the oracle's orthogonaliser (Alg. 1/2 'Orthogonalize'; P:260 reduced QR)."""
import numpy as np
import pytest

from conftest import golden
from oracle import orthogonalize, DegenerateFactor, rng


def _householder_q(A):
    """LAPACK Householder QR (numpy) with column signs fixed to R_kk > 0."""
    Q, R = np.linalg.qr(A, mode="reduced")
    s = np.sign(np.diag(R))
    s[s == 0] = 1
    return Q * s


def test_spec_examples():
    g = golden("spec_examples.json")
    I3 = np.array(g["orth_identity3"], dtype=float)
    np.testing.assert_allclose(orthogonalize(I3), I3, atol=1e-15)
    col = np.array(g["orth_column_in"], dtype=float)[:, None]
    np.testing.assert_allclose(orthogonalize(col)[:, 0], g["orth_column_out"], atol=1e-15)


@pytest.mark.parametrize("rows,r", [(6, 3), (257, 4), (1000, 32), (33, 33)])
def test_matches_householder_and_is_qr(rows, r):
    A = np.random.default_rng(rows * 100 + r).standard_normal((rows, r))
    Q = orthogonalize(A)
    np.testing.assert_allclose(Q.T @ Q, np.eye(r), atol=1e-13)
    R = Q.T @ A
    assert np.all(np.diag(R) > 0)                      # R_kk > 0 (reading C5)
    np.testing.assert_allclose(np.tril(R, -1), 0, atol=1e-11)   # upper triangular
    np.testing.assert_allclose(Q @ R, A, atol=1e-11)
    np.testing.assert_allclose(Q, _householder_q(A), atol=1e-11)


def test_ill_conditioned_twice_is_enough():
    rs = np.random.default_rng(7)
    U, _ = np.linalg.qr(rs.standard_normal((500, 8)))
    V, _ = np.linalg.qr(rs.standard_normal((8, 8)))
    A = U @ np.diag(np.logspace(0, -5, 8)) @ V.T          # kappa = 1e5
    Q = orthogonalize(A)
    assert np.abs(Q.T @ Q - np.eye(8)).max() < 1e-12
    np.testing.assert_allclose(Q, _householder_q(A), atol=1e-6)


def test_idempotent():
    A = np.random.default_rng(3).standard_normal((40, 5))
    Q = orthogonalize(A)
    np.testing.assert_allclose(orthogonalize(Q), Q, atol=1e-14)


def test_degenerate_column_repair():
    rs = np.random.default_rng(5)
    a0 = rs.standard_normal(50)
    A = np.stack([a0, np.zeros(50), 2.0 * a0, rs.standard_normal(50)], axis=1)
    with pytest.raises(DegenerateFactor):
        orthogonalize(A)
    fill = lambda k: rng.gaussian_column(9, rng.TAG_DEGENERATE, 1, 2, k, 50)
    Q = orthogonalize(A, fill)
    np.testing.assert_allclose(Q.T @ Q, np.eye(4), atol=1e-13)
    # column space = span(a0, z1, z2, a3): the QR of the repaired matrix
    Ar = A.copy()
    Ar[:, 1] = fill(1)
    Ar[:, 2] = fill(2)
    np.testing.assert_allclose(Q, _householder_q(Ar), atol=1e-10)


def test_all_zero_factor_becomes_orthonormal_random():
    fill = lambda k: rng.gaussian_column(1, rng.TAG_DEGENERATE, 0, 0, k, 20)
    Q = orthogonalize(np.zeros((20, 3)), fill)
    Z = np.stack([fill(k) for k in range(3)], axis=1)
    np.testing.assert_allclose(Q, _householder_q(Z), atol=1e-12)


def test_non_finite_rejected():
    A = np.ones((4, 2))
    A[1, 1] = np.nan
    with pytest.raises(ValueError):
        orthogonalize(A)
