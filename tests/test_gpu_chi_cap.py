"""Bond dimensions above 1024: the reference SVD has no cap (svd.hpp:79-110,
max_rank defaults to kUnbounded; gate_apply.hpp:35-38), so neither may the
GPU path. The per-gate singular-value sorts hold up to 16384 keys in one
CTA's shared memory (bond dimensions up to 8192)."""
import numpy as np
import pytest

from tests.helpers import phase_aligned_max_deviation

pytestmark = pytest.mark.gpu


@pytest.mark.slow
def test_svd_of_a_4096_vector_operand(gpu, oracle):
    """mpsim_gpu_svd of a 4096 x 4096 complex matrix with a graded spectrum
    (10 decades): singular values against LAPACK (numpy, threaded) to 1e-12
    of sigma_max, the reconstruction and the isometries to 1e-12, and the
    truncation rule on the GPU values equal to the oracle's rule on LAPACK's."""
    n = 4096
    rng = np.random.default_rng(4096)

    def haar(k):
        z = rng.standard_normal((k, k)) + 1j * rng.standard_normal((k, k))
        q, r = np.linalg.qr(z)
        return q * (np.diag(r) / np.abs(np.diag(r)))
    s_true = np.logspace(0, -10, n)
    a = (haar(n) * s_true) @ haar(n).conj().T
    u, s, vd, w = gpu.mps.svd(a)
    ref = np.linalg.svd(a, compute_uv=False)
    assert len(s) == n
    assert np.max(np.abs(s - ref)) <= 1e-12 * ref[0]
    rec = (u * s) @ vd
    assert np.max(np.abs(rec - a)) <= 1e-12 * ref[0]
    assert np.max(np.abs(u.conj().T @ u - np.eye(n))) <= 1e-12
    for cap, cutoff in ((1500, 0.0), (None, 1e-12)):
        _, s2, _, w2 = gpu.mps.svd(a, max_rank=cap, cutoff=cutoff)
        k_ref, w_ref = oracle.truncation_rank(ref, cap, cutoff)
        assert len(s2) == k_ref
        assert abs(w2 - w_ref) <= 1e-10 * w_ref


@pytest.mark.slow
def test_unbounded_22_qubit_brickwork_matches_statevector(gpu, oracle):
    """An unbounded (max_bond = kUnbounded, cutoff 0) 22-qubit Haar brickwork
    of depth 12: the centre bond grows past 1024 (theta up to 4096 x 4096);
    the MPS equals the dense statevector within 1e-10."""
    n, depth = 22, 12
    c = oracle.Circuit.brickwork(n, depth, 2202, haar=True)
    fused = c.fuse()
    g = gpu.MpsState(n, chi_hint=64)
    r = gpu.execute(g, [(q0, q1, m) for (q0, q1, _f, m) in fused.gates()], None, 0.0)
    assert r["peak_bond"] > 1024
    b = g.bond_dims()
    assert all(b[i] <= min(2 ** i, 2 ** (n - i)) for i in range(n + 1))
    sv = c.statevector()
    got = g.to_statevector(max_qubits=n)
    assert phase_aligned_max_deviation(sv, got) <= 1e-10
