"""The reference's acceptance criteria (tests/acceptance.cpp) on the GPU path,
same seeds and engine draw order as the reference binary:

  C3 oracle_equivalence     acceptance.cpp:119-145  200 random circuits, both
                                                    non-local methods, <= 1e-10
  C5 sampling_correctness   acceptance.cpp:173-241  GHZ(4) 5 sigma, chi^2 fit,
                                                    memo on/off identical
  C6 truncation_fidelity    acceptance.cpp:245-269  fidelity^2 = 1 - w (1e-9)
  C9 canonical_invariants   acceptance.cpp:346-387  isometry defects <= 1e-11

Every case is also compared with the CPU oracle on the same inputs (kept
ranks exactly, discarded weights / counts as the oracle gives them)."""
import math

import numpy as np
import pytest

from tests.helpers import MT19937_64, copy_state_to_gpu, dense_apply_2q, gate_tuples, phase_aligned_max_deviation

pytestmark = pytest.mark.gpu


def test_c3_oracle_equivalence_200_circuits(gpu, oracle):
    """acceptance.cpp:119-145: n in 2..10, 10..24 primitive ops (40 % cx/cz/swap,
    non-local allowed), unbounded policy, Swap and BondProp, against the dense
    statevector oracle. (Kept ranks are not compared here: these Clifford+T
    circuits at cutoff 0 leave exactly rank-deficient thetas whose zero
    singular values come out as exact zeros or ~1e-17 noise depending on the
    SVD, DESIGN.md §2 / SURVEY P1; the reference criterion is the state.)"""
    engine = MT19937_64(20260809)
    worst = 0.0
    for trial in range(200):
        n = 2 + engine() % 9
        gates = 10 + engine() % 15
        c = oracle.Circuit.random(n, gates, engine(), nonlocal_=True)
        fused = c.fuse()
        assert len(fused) <= 40  # fused gate budget
        sv = c.statevector()
        for bondprop in (False, True):
            g = gpu.MpsState(n)
            rg = gpu.execute(g, gate_tuples(fused), None, 0.0, bondprop=bondprop)
            dev = phase_aligned_max_deviation(sv, g.to_statevector())
            worst = max(worst, dev)
            assert dev <= 1e-10, (trial, bondprop, dev)
            n2q = sum(1 for q0, q1, _ in gate_tuples(fused) if q1 >= 0)
            assert (rg["svd_count"] > 0).sum() == n2q
    assert worst <= 1e-10


def test_c5_ghz4_corner_strings(gpu, oracle):
    """acceptance.cpp:175-193: 1e5 shots of GHZ(4), seed 97531."""
    s = gpu.MpsState(4)
    o = oracle.MpsState(4)
    for st in (s, o):
        st.apply_1q(np.array([[1, 1], [1, -1]]) / np.sqrt(2), 0)
    cx = np.eye(4, dtype=complex)[[0, 1, 3, 2]]
    for i in range(3):
        s.apply_2q_local(cx, i)
        o.apply_2q_local(cx, i)
    shots = 100000
    counts = gpu.sample(s, shots, 97531)
    assert set(counts) <= {"0000", "1111"}
    sigma = math.sqrt(shots * 0.25)
    for key in ("0000", "1111"):
        assert abs(counts.get(key, 0) - 50000.0) <= 5.0 * sigma
    assert counts == oracle.Sampler(o).sample(shots, 97531)


def test_c5_chi2_fit_random_state(gpu, oracle):
    """acceptance.cpp:195-230: random_mps(5, 4, 8675309), 2e5 shots, seed 24680,
    chi^2 goodness of fit against |amplitude|^2 (bins with expectation < 5
    pooled), p > 0.001; counts equal the oracle sampler's."""
    from scipy.stats import chi2 as chi2_dist
    o = oracle.MpsState.random(5, 4, 8675309)
    g = copy_state_to_gpu(gpu, o, chi_hint=4)
    sv = g.to_statevector()
    shots = 200000
    counts = gpu.sample(g, shots, 24680)
    stat, bins, rest_e, rest_o = 0.0, 0, 0.0, 0.0
    for b in range(32):
        bits = format(b, "05b")
        e = abs(sv[b]) ** 2 * shots
        ob = counts.get(bits, 0)
        if e < 5.0:
            rest_e += e
            rest_o += ob
            continue
        stat += (ob - e) ** 2 / e
        bins += 1
    if rest_e > 0:
        stat += (rest_o - rest_e) ** 2 / rest_e
        bins += 1
    assert chi2_dist.sf(stat, bins - 1) > 0.001
    assert counts == oracle.Sampler(o).sample(shots, 24680)


def test_c5_memo_on_off_identical(gpu, oracle):
    """acceptance.cpp:232-240: random_mps(5, 4, 1122), 20000 shots, seed 555."""
    o = oracle.MpsState.random(5, 4, 1122)
    g = copy_state_to_gpu(gpu, o, chi_hint=4)
    a = gpu.sample(g, 20000, 555)
    b = gpu.sample(g, 20000, 555, memoize=False)
    assert a == b == oracle.Sampler(o).sample(20000, 555)


def test_c6_truncation_fidelity(gpu, oracle):
    """acceptance.cpp:245-269: 12 trials, n in 4..8, centre moved to q, a Haar
    gate under max_bond 1 or 2: |<dense|mps>|^2 = 1 - w within 1e-9."""
    engine = MT19937_64(13579)
    for trial in range(12):
        n = 4 + engine() % 5
        q = engine() % (n - 1)
        o = oracle.MpsState.random(n, 8, engine())
        g = copy_state_to_gpu(gpu, o, chi_hint=8)
        g.move_center(q)
        o.move_center(q)
        pre = g.to_statevector()
        u = oracle.haar_unitary(4, engine())
        dense = dense_apply_2q(pre, u, q, q + 1, n)
        cap = 1 + engine() % 2
        rg = g.apply_2q_local(u, q, max_bond=cap, cutoff=0.0)
        ro = o.apply_2q_local(u, q, max_bond=cap, cutoff=0.0)
        f2 = abs(np.vdot(dense, g.to_statevector())) ** 2
        assert abs(f2 - (1.0 - rg.discarded_weight)) <= 1e-9, (trial, f2, rg.discarded_weight)
        assert rg.new_bond == ro.new_bond
        assert abs(rg.discarded_weight - ro.discarded_weight) <= 1e-10 * max(ro.discarded_weight, 1e-300)


def test_c9_canonical_invariants_50_states(gpu, oracle):
    """acceptance.cpp:346-387: 50 random_mps(n in 3..8, 8) states; after
    left_canonicalize every site but the last is a left isometry, after
    right_canonicalize every site but the first a right isometry (defect <=
    1e-11), and the statevector survives both (<= 1e-11); bond dims equal the
    oracle's (QR may shrink bonds, mps.cpp:57-95)."""
    engine = MT19937_64(1029384756)
    for trial in range(50):
        n = 3 + engine() % 6
        o = oracle.MpsState.random(n, 8, engine())
        g = copy_state_to_gpu(gpu, o, chi_hint=8)
        ref = g.to_statevector()
        g.left_canonicalize()
        o.move_center(n - 1)
        assert (g.bond_dims() == o.bond_dims()).all()
        for i in range(n - 1):
            t = g.site(i)
            m = t.reshape(t.shape[0] * 2, t.shape[2])
            assert np.abs(m.conj().T @ m - np.eye(t.shape[2])).max() <= 1e-11, (trial, i)
        assert phase_aligned_max_deviation(ref, g.to_statevector()) <= 1e-11
        g.right_canonicalize()
        o.move_center(0)
        assert (g.bond_dims() == o.bond_dims()).all()
        for i in range(1, n):
            t = g.site(i)
            m = t.reshape(t.shape[0], 2 * t.shape[2])
            assert np.abs(m @ m.conj().T - np.eye(t.shape[0])).max() <= 1e-11, (trial, i)
        assert phase_aligned_max_deviation(ref, g.to_statevector()) <= 1e-11
