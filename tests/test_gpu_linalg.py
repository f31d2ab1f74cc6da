"""Dense building blocks on the GPU through the C-ABI, with the reference's own
unit tests as known answers:
  qsolve             proj/tests/test_periodize.cpp:23-61
  block_lu_solve     proj/tests/test_tridiag.cpp:48-86 (synthetic systems, seeded)
plus the batched DMMA complex GEMM against numpy."""
import numpy as np
import pytest

from paper_1410_5003_b200.qpscat import SolverError, UsageError

pytestmark = pytest.mark.gpu


def rc(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (8, 8, 4), (17, 3, 5), (64, 64, 8), (81, 160, 200), (600, 600, 80),
                                   (130, 70, 33)])
def test_zgemm(gpu, M, N, K):
    rng = np.random.default_rng(M * 1000 + N)
    A, B = rc(rng, M, K), rc(rng, K, N)
    C = gpu.debug_zgemm(A, B)
    ref = A @ B
    assert np.abs(C - ref).max() <= 1e-14 * max(1.0, np.abs(ref).max()) * np.sqrt(K)


def test_qsolve_identities(gpu):
    rng = np.random.default_rng(1)
    R = rc(rng, 8, 3)
    X, r = gpu.qsolve(np.eye(8), R)
    assert np.linalg.norm(X - R) < 1e-14 and r == 8
    A = rc(rng, 20, 6)
    Q = np.linalg.qr(A)[0]
    rhs = rc(rng, 20, 4)
    assert np.linalg.norm(gpu.qsolve(Q, rhs)[0] - Q.conj().T @ rhs) < 1e-12
    B, r2 = rc(rng, 40, 20), rc(rng, 40, 5)
    pinv = np.linalg.pinv(B) @ r2
    assert np.linalg.norm(gpu.qsolve(B, r2)[0] - pinv) < 1e-12 * np.linalg.norm(pinv)
    with pytest.raises(UsageError):
        gpu.qsolve(rc(rng, 5, 8), rc(rng, 5, 2))


def test_qsolve_rank_deficient_bounded(gpu):
    rng = np.random.default_rng(11)
    Q = rc(rng, 12, 4)
    Q[:, 1] = Q[:, 0]
    rhs = rc(rng, 12, 2)
    X, r = gpu.qsolve(Q, rhs)
    assert r == 3 and np.all(np.isfinite(X))
    Qr = Q[:, [0, 2, 3]]
    Xr = np.linalg.lstsq(Qr, rhs, rcond=None)[0]
    assert np.linalg.norm(Q @ X - rhs) < np.linalg.norm(Qr @ Xr - rhs) + 1e-10
    # minimum-norm solution of the rank-3 problem
    assert np.linalg.norm(X - np.linalg.pinv(Q, rcond=1e-12) @ rhs) < 1e-12 * np.linalg.norm(X)


@pytest.mark.parametrize("m,p,n,defic", [(80, 60, 40, 7), (200, 81, 30, 5), (80, 80, 20, 0)])
def test_qsolve_matches_oracle(gpu, oracle, m, p, n, defic):
    rng = np.random.default_rng(m + p + defic)
    Q, R = rc(rng, m, p), rc(rng, m, n)
    for d in range(defic):
        Q[:, p - 1 - d] = Q[:, d] * (0.5 + 0.1j)
    Xg, rg = gpu.qsolve(Q, R)
    Xo, ro = oracle.qsolve(Q, R)
    assert rg == ro
    assert np.abs(Xg - Xo).max() < 1e-12 * np.abs(Xo).max()


def synthetic(I, n, coupled, seed):
    """proj/tests/test_tridiag.cpp:27-44 shape: 4 I + 0.3 N(0,1) diagonals, 0.5x couplings."""
    rng = np.random.default_rng(seed)
    wc = lambda: 4 * np.eye(n) + 0.3 * rc(rng, n, n)
    Ad = [wc() for _ in range(I)]
    Au = [0.5 * wc() if coupled else np.zeros((n, n)) for _ in range(I - 1)]
    Al = [0.5 * wc() if coupled else np.zeros((n, n)) for _ in range(I - 1)]
    f = rc(rng, n)
    return Ad, Au, Al, f


def dense(Ad, Au, Al, f):
    I, n = len(Ad), Ad[0].shape[0]
    D = np.zeros((I * n, I * n), dtype=complex)
    for j in range(I):
        D[j * n:(j + 1) * n, j * n:(j + 1) * n] = Ad[j]
    for j in range(I - 1):
        D[j * n:(j + 1) * n, (j + 1) * n:(j + 2) * n] = Au[j]
        D[(j + 1) * n:(j + 2) * n, j * n:(j + 1) * n] = Al[j]
    rhs = np.zeros(I * n, dtype=complex)
    rhs[:n] = f
    return np.linalg.solve(D, rhs).reshape(I, n)


def test_bcr_single_block(gpu):
    Ad, Au, Al, f = synthetic(1, 12, False, 21)
    eta = gpu.block_lu_solve_blocks(Ad, Au, Al, f)
    assert np.linalg.norm(Ad[0] @ eta[0] - f) < 1e-12 * np.linalg.norm(f)


def test_bcr_decoupled(gpu):
    Ad, Au, Al, f = synthetic(4, 10, False, 33)
    eta = gpu.block_lu_solve_blocks(Ad, Au, Al, f)
    assert np.linalg.norm(Ad[0] @ eta[0] - f) < 1e-12 * np.linalg.norm(f)
    for j in range(1, 4):
        assert np.linalg.norm(eta[j]) < 1e-14


@pytest.mark.parametrize("I,n,seed", [(3, 10, 44), (2, 16, 5), (7, 24, 9), (37, 40, 3), (64, 32, 12)])
def test_bcr_matches_dense(gpu, oracle, I, n, seed):
    Ad, Au, Al, f = synthetic(I, n, True, seed)
    eta = gpu.block_lu_solve_blocks(Ad, Au, Al, f)
    x = dense(Ad, Au, Al, f)
    assert np.linalg.norm(eta - x) < 1e-12 * np.linalg.norm(x)
    eo = oracle.block_lu_solve_blocks(Ad, Au, Al, f)  # the reference's block Thomas
    assert np.linalg.norm(eta - eo) < 1e-12 * np.linalg.norm(eo)


@pytest.mark.parametrize("I,bad", [(2, 1), (5, 2), (6, 4), (9, 8)])
def test_bcr_singular_names_layer(gpu, I, bad):
    Ad, Au, Al, f = synthetic(I, 8, False, 55)
    Ad[bad] = np.zeros_like(Ad[bad])
    with pytest.raises(SolverError) as e:
        gpu.block_lu_solve_blocks(Ad, Au, Al, f)
    assert e.value.layer == bad + 1
