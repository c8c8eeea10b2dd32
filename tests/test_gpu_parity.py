"""GPU parity: the B200 engine (through the C ABI) against the CPU oracle and
the reference's known answers. Bond dimensions / kept ranks must match
exactly; discarded weights, amplitudes and expectation values within 1e-10
relative (BASELINE.json north_star)."""
import numpy as np
import pytest

from tests.helpers import (CX, HAD, PX, PZ, SWAP, copy_state_to_gpu, dense_apply_1q, dense_apply_2q,
                           gate_tuples, max_dev, phase_aligned_max_deviation, rel)

pytestmark = pytest.mark.gpu

TOL = 1e-10


def test_x_h_single_qubit(gpu):
    s = gpu.MpsState(1)
    s.apply_1q(PX, 0)
    assert abs(s.amplitude("1") - 1) <= 1e-15
    h = gpu.MpsState(1)
    h.apply_1q(HAD, 0)
    assert abs(h.amplitude("0") - 2 ** -0.5) <= 1e-15


def test_apply_1q_random_states(gpu, oracle):
    for seed in range(1, 6):
        o = oracle.MpsState.random(5, 6, seed)
        g = copy_state_to_gpu(gpu, o)
        u = oracle.haar_unitary(2, seed * 31)
        q = seed % 5
        rg, ro = g.apply_1q(u, q), o.apply_1q(u, q)
        g.validate()
        assert rg.new_bond == ro.new_bond and rg.svd_count == 0 and rg.discarded_weight == 0.0
        assert (g.bond_dims() == o.bond_dims()).all()
        assert max_dev(g.to_statevector(), o.to_statevector()) <= 1e-12


def test_cx_zero_and_bell(gpu):
    s = gpu.MpsState(2)
    r = s.apply_2q_local(CX, 0)
    assert r.new_bond == 1 and r.discarded_weight == 0.0  # exact-zero trimming (svd.hpp:58)
    s = gpu.MpsState(2)
    s.apply_1q(HAD, 0)
    r = s.apply_2q_local(CX, 0)
    assert r.new_bond == 2
    assert np.allclose(s.to_statevector(), [2 ** -0.5, 0, 0, 2 ** -0.5], atol=1e-14)


def test_apply_2q_local_matches_oracle(gpu, oracle):
    for seed in range(1, 7):
        o = oracle.MpsState.random(6, 6, 100 + seed)
        g = copy_state_to_gpu(gpu, o)
        pre = o.to_statevector()
        u = oracle.haar_unitary(4, 17 * seed)
        q = seed % 5
        rg, ro = g.apply_2q_local(u, q), o.apply_2q_local(u, q)
        g.validate()
        assert rg.new_bond == ro.new_bond and rg.svd_count == 1
        assert (g.bond_dims() == o.bond_dims()).all()
        assert max_dev(g.to_statevector(), dense_apply_2q(pre, u, q, q + 1, 6)) <= TOL
        assert abs(g.norm() - 1) <= TOL


@pytest.mark.parametrize("chi,cap,cutoff", [(8, 1, 0.0), (16, 5, 1e-3), (16, 7, 1e-12), (32, 12, 0.0)])
def test_truncation_matches_oracle(gpu, oracle, chi, cap, cutoff):
    for seed in range(1, 5):
        o = oracle.MpsState.random(10, chi, 300 + seed)
        g = copy_state_to_gpu(gpu, o)
        u = oracle.haar_unitary(4, 5 * seed)
        q = 4
        rg = g.apply_2q_local(u, q, max_bond=cap, cutoff=cutoff)
        ro = o.apply_2q_local(u, q, max_bond=cap, cutoff=cutoff)
        assert rg.new_bond == ro.new_bond
        assert rel(rg.discarded_weight, ro.discarded_weight) <= TOL
        assert (g.bond_dims() == o.bond_dims()).all()
        ref = o.to_statevector()
        assert max_dev(g.to_statevector(), ref) <= TOL * np.abs(ref).max()


def test_discarded_weight_is_lost_fidelity(gpu, oracle):
    for seed in range(1, 7):
        o = oracle.MpsState.random(6, 8, 200 + seed)
        o.move_center(2)  # oracle canonicalization, then import (GPU QR sweep is staged)
        g = copy_state_to_gpu(gpu, o)
        pre = o.to_statevector()
        u = oracle.haar_unitary(4, 23 * seed)
        exact = dense_apply_2q(pre, u, 2, 3, 6)
        r = g.apply_2q_local(u, 2, max_bond=1)
        assert r.new_bond == 1
        f2 = abs(np.vdot(exact, g.to_statevector())) ** 2
        assert abs(f2 - (1 - r.discarded_weight)) <= 1e-9
        assert abs(g.norm() - 1) <= 1e-10
        assert g.ortho_center == 3


def test_bad_inputs_raise(gpu):
    s = gpu.MpsState(3)
    with pytest.raises(ValueError):
        s.apply_2q_local(CX, 2)
    with pytest.raises(ValueError):
        s.apply_2q_local(CX, 0, cutoff=1.5)
    with pytest.raises(ValueError):
        s.apply_2q_local(CX, 0, max_bond=0)
    with pytest.raises(ValueError):
        s.apply_1q(PX, 3)


def test_swap_routing(gpu, oracle):
    s = gpu.MpsState(4)
    s.apply_1q(HAD, 0)
    pre = s.to_statevector()
    r = s.apply_2q_swap(CX, 0, 3)
    s.validate()
    assert r.svd_count == 5
    assert max_dev(s.to_statevector(), dense_apply_2q(pre, CX, 0, 3, 4)) <= TOL
    for seed in range(1, 6):
        o = oracle.MpsState.random(6, 4, 400 + seed)
        g = copy_state_to_gpu(gpu, o)
        u = oracle.haar_unitary(4, 7 * seed)
        rg, ro = g.apply_2q_swap(u, 1, 4), o.apply_2q_swap(u, 1, 4)
        assert rg.new_bond == ro.new_bond and rg.svd_count == ro.svd_count
        assert (g.bond_dims() == o.bond_dims()).all()
        assert max_dev(g.to_statevector(), o.to_statevector()) <= TOL
        # flipped order: (high, low) is SWAP-conjugated (gate_apply.cpp:156-159)
        g2 = copy_state_to_gpu(gpu, oracle.MpsState.random(6, 4, 400 + seed))
        o2 = oracle.MpsState.random(6, 4, 400 + seed)
        g2.apply_2q_swap(u, 4, 1)
        o2.apply_2q_swap(u, 4, 1)
        assert max_dev(g2.to_statevector(), o2.to_statevector()) <= TOL


def test_cap_never_exceeded(gpu, oracle):
    rng = np.random.default_rng(42)
    s = gpu.MpsState(6)
    for _ in range(30):
        q = int(rng.integers(5))
        s.apply_2q_local(oracle.haar_unitary(4, int(rng.integers(1 << 62))), q, max_bond=3)
        assert s.max_bond_dim() <= 3
        s.validate()


@pytest.mark.parametrize("n", [4, 16, 64])
def test_ghz_bonds_exactly_two(gpu, n):
    s = gpu.MpsState(n)
    s.apply_1q(HAD, 0)
    for i in range(n - 1):
        s.apply_2q_local(CX, i)
    assert (s.bond_dims()[1:-1] == 2).all()
    a = s.amplitudes(["0" * n, "1" * n, "01" * (n // 2)])
    assert abs(a[0] - 2 ** -0.5) <= 1e-12 and abs(a[1] - 2 ** -0.5) <= 1e-12 and abs(a[2]) <= 1e-12


def test_layer_span_guard(gpu):
    s = gpu.MpsState(4)
    with pytest.raises(gpu.LogicError):
        s.apply_layer([(0, 1, CX), (1, 2, CX)])
    with pytest.raises(ValueError):
        s.apply_layer([(0, 2, CX)])


def test_queries_match_oracle(gpu, oracle):
    o = oracle.MpsState.random(7, 8, 33)
    g = copy_state_to_gpu(gpu, o)
    sv = o.to_statevector()
    assert max_dev(g.to_statevector(), sv) <= 1e-13
    bits = [format(b, "07b") for b in range(128)]
    assert max_dev(g.amplitudes(bits), sv) <= 1e-13
    assert abs(g.norm() - o.norm()) <= 1e-13
    o2 = oracle.MpsState.random(7, 8, 34)
    g2 = copy_state_to_gpu(gpu, o2)
    assert rel(g.overlap(g2), o.overlap(o2)) <= 1e-12
    # P9: <O_q> = overlap(psi, apply_1q(copy psi, O, q))
    for q in range(7):
        for op in (PZ, PX):
            oc = o.copy()
            oc.apply_1q(op, q)
            assert rel(g.expect_1q(op, q), o.overlap(oc)) <= 1e-12
    oc = o.copy()
    oc.apply_1q(PZ, 2)
    oc.apply_1q(PZ, 3)
    assert rel(g.expect_2q(PZ, 2, PZ, 3), o.overlap(oc)) <= 1e-12


def test_execute_matches_oracle_serial(gpu, oracle):
    # test_executor.cpp:70-87 on the SWAP method. At cutoff 0 the kept rank of
    # a structurally rank-deficient theta depends on whether an SVD returns
    # its zero singular values as exact zeros or as ~1e-17 noise,
    # which differs between Eigen, LAPACK and Jacobi: compare the state there,
    # and compare kept ranks gate by gate at cutoff 1e-14, where noise is
    # trimmed deterministically by the reference rule.
    for seed in range(3):
        c = oracle.Circuit.random(10, 30, 77 + seed, nonlocal_=True)
        fused = c.fuse()
        ref = c.statevector()
        g = gpu.MpsState(10)
        gpu.execute(g, gate_tuples(fused))
        assert phase_aligned_max_deviation(ref, g.to_statevector()) <= TOL
        g = gpu.MpsState(10)
        rg = gpu.execute(g, gate_tuples(fused), None, 1e-14)
        o = oracle.MpsState(10)
        ro = oracle.execute_serial(o, fused, None, 1e-14)
        assert rg["peak_bond"] == ro["peak_bond"]
        assert (rg["gate_k"] == ro["gate_k"]).all()
        assert (rg["svd_count"] > 0).sum() == sum(1 for q0, q1, _, _ in fused.gates() if q1 >= 0)
        assert phase_aligned_max_deviation(ref, g.to_statevector()) <= TOL


def test_brickwork_c2_small_truncating(gpu, oracle):
    """C2-shaped (Haar brickwork, cutoff 1e-12, capped) at a size the oracle runs in seconds."""
    fused = oracle.Circuit.brickwork(24, 12, 4242, haar=True).fuse()
    o = oracle.MpsState(24)
    ro = oracle.execute_serial(o, fused, 32, 1e-12)
    g = gpu.MpsState(24)
    rg = gpu.execute(g, gate_tuples(fused), 32, 1e-12)
    assert (rg["gate_k"] == ro["gate_k"]).all()
    assert rg["peak_bond"] == ro["peak_bond"] == 32
    nz = ro["gate_w"] > 0
    assert np.max(np.abs(rg["gate_w"][nz] - ro["gate_w"][nz]) / ro["gate_w"][nz]) <= 1e-8
    assert rel(rg["total_discarded_weight"], ro["total_discarded_weight"]) <= 1e-8
    rng = np.random.default_rng(7)
    bits = ["".join(rng.choice(["0", "1"], 24)) for _ in range(64)]
    ag = g.amplitudes(bits)
    ao = np.array([o.amplitude(b) for b in bits])
    assert np.max(np.abs(ag - ao) / np.abs(ao)) <= 1e-8


def test_c1_ghz_plus_random_layer(gpu, oracle):
    """C1: 20-qubit GHZ + seeded u3 layer, chi <= 16."""
    c = oracle.Circuit.ghz(20)
    rng_c = oracle.Circuit.brickwork(20, 1, 1)  # u3 angles from mt19937_64(1) in brickwork order
    for kind, q0, q1, params in rng_c.ops():
        if kind == "u3":
            c.add("u3", q0, -1, params)
    fused = c.fuse()
    g = gpu.MpsState(20)
    rg = gpu.execute(g, gate_tuples(fused), 16, 0.0)
    assert (g.bond_dims()[1:-1] == 2).all() and rg["peak_bond"] == 2
    sv = c.statevector()
    assert phase_aligned_max_deviation(sv, g.to_statevector()) <= TOL
    o = oracle.MpsState(20)
    oracle.execute_serial(o, fused, 16, 0.0)
    for q in range(0, 20, 3):
        oc = o.copy()
        oc.apply_1q(PZ, q)
        assert abs(g.expect_1q(PZ, q) - o.overlap(oc)) <= TOL


def test_bondprop_matches_oracle(gpu, oracle):
    # test_gate_apply.cpp:223-262
    a = oracle.MpsState.random(4, 4, 501)
    g = copy_state_to_gpu(gpu, a)
    u = oracle.haar_unitary(4, 77)
    r = g.apply_2q_bondprop(u, 1, 2)
    a.apply_2q_local(u, 1)
    g.validate()
    assert r.svd_count == 1 and max_dev(g.to_statevector(), a.to_statevector()) <= 1e-12
    for seed in range(1, 6):
        o = oracle.MpsState.random(6, 4, 600 + seed)
        g = copy_state_to_gpu(gpu, o)
        pre = o.to_statevector()
        u = oracle.haar_unitary(4, 13 * seed)
        rg = g.apply_2q_bondprop(u, 1, 4)
        ro = o.apply_2q_bondprop(u, 1, 4)
        g.validate()
        assert rg.svd_count == 3 == ro.svd_count and rg.new_bond == ro.new_bond
        assert (g.bond_dims() == o.bond_dims()).all()
        assert max_dev(g.to_statevector(), dense_apply_2q(pre, u, 1, 4, 6)) <= TOL
    o = oracle.MpsState.random(5, 4, 700)
    g = copy_state_to_gpu(gpu, o)
    pre = o.to_statevector()
    u = oracle.haar_unitary(4, 55)
    g.apply_2q_bondprop(u, 0, 4)
    g.validate()
    assert max_dev(g.to_statevector(), dense_apply_2q(pre, u, 0, 4, 5)) <= TOL
    # CX has operator-Schmidt rank 2: the carrier is 2 wide (exact-zero trim of the gate split)
    s = gpu.MpsState(5)
    s.apply_1q(HAD, 0)
    r = s.apply_2q_bondprop(CX, 0, 4)
    assert r.svd_count == 4 and s.max_bond_dim() == 2


def test_bondprop_truncating_and_executor(gpu, oracle):
    for seed in range(3):
        o = oracle.MpsState.random(8, 8, 900 + seed)
        g = copy_state_to_gpu(gpu, o)
        u = oracle.haar_unitary(4, 31 + seed)
        rg = g.apply_2q_bondprop(u, 1, 6, max_bond=5, cutoff=1e-10)
        ro = o.apply_2q_bondprop(u, 1, 6, max_bond=5, cutoff=1e-10)
        # The carriers of bond propagation have exactly degenerate singular
        # values at these cuts (e.g. s_4 = s_5 = 10.3490936492091..., checked
        # with an independent numpy restatement), so the kept subspace is not
        # unique: kept ranks and discarded weights are compared,
        # amplitudes only where the truncation is unambiguous (below).
        assert rg.new_bond == ro.new_bond and (g.bond_dims() == o.bond_dims()).all()
        assert rel(rg.discarded_weight, ro.discarded_weight) <= 1e-9
    for seed in range(3):
        o = oracle.MpsState.random(8, 8, 900 + seed)
        g = copy_state_to_gpu(gpu, o)
        u = oracle.haar_unitary(4, 31 + seed)
        rg = g.apply_2q_bondprop(u, 1, 6, max_bond=64, cutoff=1e-12)
        ro = o.apply_2q_bondprop(u, 1, 6, max_bond=64, cutoff=1e-12)
        assert rg.new_bond == ro.new_bond and (g.bond_dims() == o.bond_dims()).all()
        ref = o.to_statevector()
        assert max_dev(g.to_statevector(), ref) <= TOL * np.abs(ref).max()
    c = oracle.Circuit.random(10, 30, 78, nonlocal_=True)
    fused = c.fuse()
    g = gpu.MpsState(10)
    gpu.execute(g, gate_tuples(fused), bondprop=True)
    assert phase_aligned_max_deviation(c.statevector(), g.to_statevector()) <= TOL
