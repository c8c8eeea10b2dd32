"""The GPU truncated SVD (the batched one-sided Jacobi kernels behind
mpsim_gpu_svd) against the reference SVD contract, test_tensor.cpp:232-364,
and against the CPU oracle (LAPACK zgesdd) on seeded matrices."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rand(rng, r, c):
    return rng.standard_normal((r, c)) + 1j * rng.standard_normal((r, c))


def test_identity_and_diagonal(gpu):
    _, s, _, w = gpu.mps.svd(np.eye(2))
    assert len(s) == 2 and np.allclose(s, 1, atol=1e-14) and w == 0.0
    _, s, _, _ = gpu.mps.svd(np.diag([3.0, 4.0]))
    assert abs(s[0] - 4) < 1e-13 and abs(s[1] - 3) < 1e-13


@pytest.mark.parametrize("shape", [(6, 5), (5, 6), (2, 2), (1, 7), (7, 1), (33, 17), (40, 64), (130, 129),
                                   (129, 200), (256, 160)])
def test_reconstruct_isometric_sorted(gpu, shape):
    rng = np.random.default_rng(23)
    for _ in range(4):
        m = _rand(rng, *shape)
        u, s, vd, w = gpu.mps.svd(m)
        k = len(s)
        assert k == min(shape) and w == 0.0
        assert np.linalg.norm(u @ np.diag(s) @ vd - m) / np.linalg.norm(m) <= 1e-12
        # One factor is the converged Jacobi operand (orthonormal to the
        # Jacobi tolerance); the other is contracted from A (V^dag = S^-1 U^H A,
        # or U = A V S^-1 when the sweeps ran on the QR-preconditioned A^H
        # side) and inherits that residual amplified by (s_max / s_i)(s_max /
        # s_j). The reference's own case (6x5, test_tensor.cpp:247-277) meets
        # 1e-12 on both. The operand side is orthonormalised before the split
        # (split.cu), so it is orthonormal to rounding.
        kappa2 = (s[0] / s[-1]) ** 2
        eu = np.abs(u.conj().T @ u - np.eye(k)).max()
        ev = np.abs(vd @ vd.conj().T - np.eye(k)).max()
        assert min(eu, ev) <= 2e-14, (shape, eu, ev)
        assert max(eu, ev) <= 1e-12 * max(1.0, kappa2 / 100)
        assert np.all(np.diff(s) <= 0) and s[-1] >= 0
        assert np.abs(s - np.linalg.svd(m, compute_uv=False)).max() <= 1e-13 * s[0]


def test_discarded_weight_vs_eigensolver(gpu):
    rng = np.random.default_rng(29)
    m = _rand(rng, 8, 6)
    ev = np.linalg.eigvalsh(m.conj().T @ m)
    u, s, vd, w = gpu.mps.svd(m, 3, 0.0)
    assert len(s) == 3
    assert abs(w - ev[:3].sum() / ev.sum()) <= 1e-12
    err2 = np.linalg.norm(u @ np.diag(s) @ vd - m) ** 2
    assert abs(err2 / np.linalg.norm(m) ** 2 - w) <= 1e-12


def test_cutoff_rule(gpu):
    _, s, _, w = gpu.mps.svd(np.array([[1, 0], [0, 0]], dtype=complex), None, 0.0)
    assert len(s) == 1 and w == 0.0  # exact zero trimmed at cutoff 0
    _, s, _, w = gpu.mps.svd(np.diag([1.0, 0.1]), None, 0.5)
    assert len(s) == 1 and abs(w - 0.01 / 1.01) <= 1e-14
    _, s, _, _ = gpu.mps.svd(np.diag([1.0, 0.1]), None, 0.001)
    assert len(s) == 2
    _, s, _, w = gpu.mps.svd(np.zeros((3, 2)))
    assert len(s) == 1 and s[0] == 0.0 and w == 0.0
    # rank-1 with duplicated columns: the zero singular value is exact
    _, s, _, _ = gpu.mps.svd(np.array([[1, 1], [0, 0]], dtype=complex) / np.sqrt(2), None, 0.0)
    assert len(s) == 1 and abs(s[0] - 1) < 1e-15


def test_bad_options(gpu):
    with pytest.raises(ValueError):
        gpu.mps.svd(np.eye(2), 0, 0.0)
    with pytest.raises(ValueError):
        gpu.mps.svd(np.eye(2), 1, 1.0)
    # (no size cap below the sort capacity of 16384 vectors: an all-zero
    # 2100 x 2100 operand, once rejected, is a rank-1 result now)
    _, s, _, w = gpu.mps.svd(np.zeros((2100, 2100)), 4, 0.0)
    assert len(s) == 1 and s[0] == 0.0 and w == 0.0


@pytest.mark.parametrize("cap,cutoff", [(None, 1e-12), (9, 0.0), (20, 1e-6), (1, 0.0)])
def test_kept_rank_matches_oracle(gpu, oracle, cap, cutoff):
    rng = np.random.default_rng(31)
    for trial in range(6):
        r, c = [(48, 48), (64, 32), (32, 64), (96, 80), (20, 100), (128, 128)][trial]
        # graded spectrum so the cutoff bites
        a = _rand(rng, r, c) * np.logspace(0, -9, c)[None, :]
        _, sg, _, wg = gpu.mps.svd(a, cap, cutoff)
        _, so, _, wo = oracle.svd(a, cap, cutoff)
        assert len(sg) == len(so)
        assert np.abs(sg - so).max() <= 1e-13 * so[0]
        assert abs(wg - wo) <= 1e-10 * max(wo, 1e-300) or abs(wg - wo) < 1e-15


@pytest.mark.parametrize("shape", [(200, 200), (160, 300)])
def test_rank_deficient_preconditioned(gpu, shape):
    """Low-rank operands on the QR-preconditioned path (n >= 128): exact zero
    Householder columns, zero rows of R, noise-floor vectors."""
    rng = np.random.default_rng(31)
    m = _rand(rng, shape[0], 3) @ _rand(rng, 3, shape[1])
    u, s, vd, w = gpu.mps.svd(m, None, 1e-14)
    ref = np.linalg.svd(m, compute_uv=False)
    assert len(s) == 3
    assert np.abs(s - ref[:3]).max() <= 1e-13 * ref[0]
    assert np.linalg.norm(u @ np.diag(s) @ vd - m) / np.linalg.norm(m) <= 1e-12


def test_random_shapes_fuzz(gpu):
    """Seeded fuzz over shapes 1..300 x 1..300 (both sides of the QR
    preconditioning threshold, odd and ragged sizes, tall and wide): singular
    values against numpy's LAPACK to 1e-12 relative to s_max, reconstruction
    to 1e-12, and the kept rank / discarded weight of a cap + cutoff policy
    against the reference rule applied to numpy's values."""
    rng = np.random.default_rng(2601)
    for _ in range(24):
        r, c = (int(x) for x in rng.integers(1, 301, size=2))
        # graded spectra exercise the relative-accuracy path
        a = _rand(rng, r, c) * np.logspace(0, -int(rng.integers(0, 9)), c)[None, :]
        u, s, vd, w = gpu.mps.svd(a)
        ref = np.linalg.svd(a, compute_uv=False)
        assert len(s) == min(r, c)
        assert np.abs(s - ref).max() <= 1e-12 * ref[0], (r, c)
        assert np.linalg.norm(u @ np.diag(s) @ vd - a) <= 1e-12 * np.linalg.norm(a), (r, c)
        cap = int(rng.integers(1, min(r, c) + 1))
        _, s2, _, w2 = gpu.mps.svd(a, max_rank=cap, cutoff=1e-6)
        tot = float((ref ** 2).sum())
        keep, tail = len(ref), 0.0
        while keep > 1 and tail + ref[keep - 1] ** 2 <= 1e-6 * tot:  # svd.hpp:48-74
            tail += ref[keep - 1] ** 2
            keep -= 1
        keep = min(keep, cap)
        assert len(s2) == keep, (r, c, cap)
        assert abs(w2 - float((ref[keep:] ** 2).sum()) / tot) <= 1e-10 * max(w2, 1e-300) + 1e-15, (r, c)


@pytest.mark.parametrize("gap", [0.7, 0.07])
def test_truncated_subspace_at_lapack_accuracy(gpu, gap):
    """The kept left subspace of a truncating SVD (2048 x 2048, keep 1024 of a
    smooth spectrum with a relative gap `gap` at the cut) within 1e-12 / gap of
    numpy's LAPACK, and the truncated product U S V^dag within 1e-13 (the
    accuracy the C4 window needs; that window's own truncating thetas, which
    the old quadratic-phase exit left at 4.4e-11 / 2.3e-9, are exercised by
    tests/test_gpu_golden.py)."""
    rng = np.random.default_rng(20261019)
    n, k = 2048, 1024
    s = np.concatenate([np.linspace(1.0, 0.3, k), (1.0 - gap) * 0.3 * np.linspace(1.0, 1e-3, n - k)])
    q1 = np.linalg.qr(_rand(rng, n, n))[0]
    q2 = np.linalg.qr(_rand(rng, n, n))[0]
    th = (q1 * s) @ q2.conj().T
    u, sg, vd, w = gpu.mps.svd(th, max_rank=k)
    un, sn, vn = np.linalg.svd(th)
    assert len(sg) == k
    assert abs(w - float((sn[k:] ** 2).sum() / (sn ** 2).sum())) <= 1e-12 * w
    d = np.linalg.norm(u @ u.conj().T - un[:, :k] @ un[:, :k].conj().T, 2)
    assert d <= 1e-12 / gap, d
    prod = u @ (sg[:, None] * vd) - (un[:, :k] * sn[:k]) @ vn[:k]
    assert np.linalg.norm(prod) <= 1e-13 * np.linalg.norm(th)
