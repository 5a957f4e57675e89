"""Per-cluster dense kernels through the C ABI (h2f_dense_*), every
implementation the factorization dispatches to by size, at the sizes the
upper levels of the BASELINE configs reach.  The CPU
reference is LAPACK through NumPy, i.e. the calls the reference makes
(factorization.py:78-99)."""
import numpy as np
import pytest

from paper_2509_11152_b200 import _lib

pytestmark = pytest.mark.gpu


def graded(m, n, decay, seed):
    """m x n with singular values 10**(-decay * i / m), random singular vectors."""
    rng = np.random.Generator(np.random.Philox(seed))
    u, _ = np.linalg.qr(rng.standard_normal((m, m)))
    v, _ = np.linalg.qr(rng.standard_normal((n, m)))
    sig = 10.0 ** (-decay * np.arange(m) / max(m, 1))
    return (u * sig) @ v.T, sig


@pytest.mark.parametrize("n,path", [(40, 0), (130, 0), (40, 1), (130, 1), (300, 1), (700, 1), (130, 2), (300, 2)])
def test_jacobi_svd_matches_lapack(n, path):
    # R is the triangular factor the augmentation feeds in (factorization.py:78-79)
    Y, sig = graded(n, 3 * n, 12.0, n + path)
    R = np.linalg.qr(Y.T, mode="r")
    # threshold in the middle of a singular-value gap (the kept count is exact)
    thresh = np.sqrt(sig[n // 3] * sig[n // 3 + 1])
    U, kept, sweeps, ms = _lib.dense_svd(R, thresh, path)
    u_ref, s_ref, _ = np.linalg.svd(R.T)
    assert kept == int(np.sum(s_ref >= thresh)) == n // 3 + 1
    # left singular vectors up to sign (simple spectrum)
    dots = np.abs(np.sum(U * u_ref[:, :kept].T, axis=1))
    assert np.max(np.abs(dots - 1.0)) < 1e-10
    if path:
        assert 1 <= sweeps < 60


@pytest.mark.parametrize("n,wf,path", [(30, 2000, 0), (120, 5000, 0), (30, 2000, 1), (120, 5000, 1),
                                       (300, 9000, 1), (500, 700, 1), (200, 150, 1)])
def test_qr_r_matches_lapack(n, wf, path):
    Y, _ = graded(n, wf, 6.0, n + wf) if n <= wf else (None, None)
    if Y is None:
        Y = np.random.Generator(np.random.Philox(n)).standard_normal((n, wf))
    R, ms = _lib.dense_qr_r(Y, path)
    R_ref = np.linalg.qr(Y.T, mode="r")
    if path == 1:
        # same Householder conventions (dlarfg): R itself agrees
        assert np.linalg.norm(R - R_ref) <= 1e-12 * np.linalg.norm(R_ref)
    else:
        # the shared-memory TSQR folds chunks: R agrees up to row signs
        d = np.sign(np.diag(R)) * np.sign(np.diag(R_ref))
        assert np.linalg.norm(d[:, None] * R - R_ref) <= 1e-12 * np.linalg.norm(R_ref)


@pytest.mark.parametrize("s,kt,path", [(64, 20, 0), (200, 120, 0), (64, 20, 1), (200, 120, 1), (900, 600, 1),
                                       (300, 0, 1), (150, 150, 1)])
def test_complement_matches_lapack(s, kt, path):
    rng = np.random.Generator(np.random.Philox(s + kt))
    b_aug = np.linalg.qr(rng.standard_normal((s, max(kt, 1))))[0][:, :kt]
    Q, ms = _lib.dense_complement(np.ascontiguousarray(b_aug.T), path)
    r = s - kt
    assert np.array_equal(Q[:, r:], b_aug)                      # trailing columns are b_aug itself
    assert np.linalg.norm(Q.T @ Q - np.eye(s)) <= 1e-12 * s     # orthogonal
    if kt:
        q_ref, _ = np.linalg.qr(b_aug, mode="complete")         # factorization.py:98
        assert np.linalg.norm(Q[:, :r] - q_ref[:, kt:]) <= 1e-11 * np.sqrt(s)
