"""BASELINE.json configs C3-C5 as GPU-vs-oracle parity runs,
shaped so the CPU oracle finishes in seconds: the same fused gate lists go
through the GPU executor and the oracle's execute_parallel / execute_serial.
Checks are those the table names: per-gate kept ranks exactly, discarded
weights and amplitudes / expectation values to 1e-10 relative."""
import numpy as np
import pytest

from tests.helpers import gate_tuples, rel

pytestmark = pytest.mark.gpu

PZ = np.diag([1.0, -1.0]).astype(np.complex128)
PX = np.array([[0, 1], [1, 0]], dtype=np.complex128)


def _amplitude_parity(g, o, n, seed, count=16, tol=1e-10, zero=0.0):
    """Relative parity of random amplitudes; amplitudes below `zero` (structural
    zeros of CX-built states, ~1e-19 .. 1e-35 in either code) only have to be
    below it on both sides."""
    rng = np.random.default_rng(seed)
    bits = ["".join(rng.choice(["0", "1"], n)) for _ in range(count)]
    ag = g.amplitudes(bits)
    ao = np.array([o.amplitude(b) for b in bits])
    big = np.abs(ao) > zero
    assert big.any()
    assert np.max(np.abs(ag[big] - ao[big]) / np.abs(ao[big])) <= tol
    assert (np.abs(ag[~big]) <= 10 * max(zero, 1e-300)).all()


@pytest.mark.slow
def test_c5_wide_shallow_brickwork(gpu, oracle):
    """C5: 1000-qubit Haar brickwork depth 10 at chi=128, cutoff 1e-12: ~500
    disjoint gates per layer in one batched launch sequence (layer batching)."""
    n = 1000
    fused = oracle.Circuit.brickwork(n, 10, 1000, haar=True).fuse()
    o = oracle.MpsState(n)
    ro = oracle.execute_parallel(o, fused, 128, 1e-12, workers=16)
    g = gpu.MpsState(n, chi_hint=128)
    rg = gpu.execute(g, gate_tuples(fused), 128, 1e-12)
    assert (rg["gate_k"] == ro["gate_k"]).all()
    assert (g.bond_dims() == o.bond_dims()).all()
    assert rg["peak_bond"] == ro["peak_bond"] == 128
    nz = ro["gate_w"] > 0
    assert np.max(np.abs(rg["gate_w"][nz] - ro["gate_w"][nz]) / ro["gate_w"][nz]) <= 1e-10
    assert rel(rg["total_discarded_weight"], ro["total_discarded_weight"]) <= 1e-10
    _amplitude_parity(g, o, n, 7)


@pytest.mark.slow
def test_c3_brickwork_with_nonadjacent_gates(gpu, oracle):
    """C3-shaped: Haar brickwork in which every 4th pair of each entangling layer
    is replaced by a CX over distance 2..4 (SWAP-routed, decompose_nonlocal
    order), truncating at chi=16 so SWAP gates truncate too (P6)."""
    n, depth, chi = 24, 8, 16
    c = oracle.Circuit(n)
    rng = np.random.default_rng(2601)
    for layer in range(depth):
        for i, p in enumerate(range(layer % 2, n - 1, 2)):
            if i % 4 == 3:
                d = 2 + int(rng.integers(3))
                if p + d < n:
                    c.add("cx", p, p + d)
                    continue
            z = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
            q, r = np.linalg.qr(z)
            c.add("u4", p, p + 1, matrix=q * (np.diag(r) / np.abs(np.diag(r))))
    fused = c.fuse()
    o = oracle.MpsState(n)
    ro = oracle.execute_serial(o, fused, chi, 1e-12)
    g = gpu.MpsState(n, chi_hint=chi)
    rg = gpu.execute(g, gate_tuples(fused), chi, 1e-12)
    assert (rg["gate_k"] == ro["gate_k"]).all()
    # a CX over distance d is 2(d-1)+1 truncating SVDs (gate_apply.cpp:149-179)
    assert rg["svd_count"].max() >= 3
    assert (g.bond_dims() == o.bond_dims()).all()
    assert rg["peak_bond"] == ro["peak_bond"] == chi
    # CX gates leave exactly rank-deficient thetas: discarded weights at the
    # rounding-noise level (~1e-30 from LAPACK, 0 or ~1e-25 here: sigma^2 <=
    # (64 eps)^2 ||theta||^2 snaps to 0, P1) carry no information;
    # compare the weights above 1e-16 (the cutoff is 1e-12)
    floor = 1e-16
    nz = ro["gate_w"] > floor
    assert nz.sum() > 0  # the cap truncates
    assert np.max(np.abs(rg["gate_w"][nz] - ro["gate_w"][nz]) / ro["gate_w"][nz]) <= 1e-10
    assert (rg["gate_w"][~nz] <= floor).all()
    _amplitude_parity(g, o, n, 11, count=64, zero=1e-12)


@pytest.mark.slow
def test_c4_tfim_trotter_expectations(gpu, oracle):
    """C4-shaped: disordered non-Clifford TFIM Trotter steps (cx; rz; cx on even
    then odd bonds, rx on every site; J dt = 0.8, h_i dt = 0.8 + 0.2 (u_i - 1/2))
    under chi=1024, cutoff 1e-12; <Z_i>, <X_i> against the P9 oracle
    definition overlap(psi, apply_1q(psi, O, i))."""
    n, steps = 16, 6
    c = oracle.Circuit(n)
    u = np.random.default_rng(256).random(n)
    jdt = 0.8
    for _ in range(steps):
        for parity in (0, 1):
            for p in range(parity, n - 1, 2):
                c.add("cx", p, p + 1)
                c.add("rz", p + 1, -1, (-2 * jdt,))
                c.add("cx", p, p + 1)
        for q in range(n):
            c.add("rx", q, -1, (-2 * (0.8 + 0.2 * (u[q] - 0.5)),))
    fused = c.fuse()
    o = oracle.MpsState(n)
    ro = oracle.execute_serial(o, fused, 1024, 1e-12)
    g = gpu.MpsState(n, chi_hint=256)
    rg = gpu.execute(g, gate_tuples(fused), 1024, 1e-12)
    assert (rg["gate_k"] == ro["gate_k"]).all()
    assert (g.bond_dims() == o.bond_dims()).all()
    for q in range(n):
        for op in (PZ, PX):
            oc = o.copy()
            oc.apply_1q(op, q)
            ref = o.overlap(oc).real
            got = g.expect_1q(op, q).real
            assert abs(got - ref) <= 1e-10 * max(1.0, abs(ref)), (q, got, ref)
    # amplitudes of this 16-qubit state are ~2^-8: after 180 gates the rounding
    # of two different SVDs differs by a few 1e-13 absolute, so the relative
    # check on single amplitudes gets 1e-9 (the C4 checks are the expectations)
    _amplitude_parity(g, o, n, 3, tol=1e-9)
