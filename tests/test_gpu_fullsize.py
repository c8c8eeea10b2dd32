"""Parity at the BASELINE sizes: chi = 512 (C3 / headline metric) and chi = 1024
(C4) gates, GPU against the CPU oracle on identical seeded inputs, plus
size-independent properties of a full layer."""
import numpy as np
import pytest

from tests.helpers import copy_state_to_gpu, rel

pytestmark = pytest.mark.gpu


def _fullsize(gpu, oracle, n, chi, seed, qs, cutoff=1e-12):
    o = oracle.MpsState.random(n, chi, seed)
    g = copy_state_to_gpu(gpu, o, chi_hint=chi)
    for i, q in enumerate(qs):
        u = oracle.haar_unitary(4, seed + 31 * i)
        assert o.bond_dims()[q] == o.bond_dims()[q + 1] == o.bond_dims()[q + 2] == chi
        rg = g.apply_2q_local(u, q, max_bond=chi, cutoff=cutoff)
        ro = o.apply_2q_local(u, q, max_bond=chi, cutoff=cutoff)
        assert rg.new_bond == ro.new_bond == chi
        assert rel(rg.discarded_weight, ro.discarded_weight) <= 1e-10
    assert (g.bond_dims() == o.bond_dims()).all()
    rng = np.random.default_rng(7)
    bits = ["".join(rng.choice(["0", "1"], n)) for _ in range(16)]
    ag = g.amplitudes(bits)
    ao = np.array([o.amplitude(b) for b in bits])
    assert np.max(np.abs(ag - ao) / np.abs(ao)) <= 1e-10
    return g, o


@pytest.mark.slow
def test_chi512_gates_match_oracle(gpu, oracle):
    _fullsize(gpu, oracle, 24, 512, 2601, [10, 12])


@pytest.mark.slow
def test_chi512_ragged_gates_match_oracle(gpu, oracle):
    """Gates where 2Dl != 2Dr (theta 512 x 1024 and 1024 x 512 at the chain's
    growing edge): both QR-preconditioned factor formulas."""
    n, chi, seed = 24, 512, 77
    o = oracle.MpsState.random(n, chi, seed)
    g = copy_state_to_gpu(gpu, o, chi_hint=chi)
    for i, q in enumerate([8, 14]):
        u = oracle.haar_unitary(4, seed + 17 * i)
        rg = g.apply_2q_local(u, q, max_bond=chi, cutoff=1e-12)
        ro = o.apply_2q_local(u, q, max_bond=chi, cutoff=1e-12)
        assert rg.new_bond == ro.new_bond
        assert rel(rg.discarded_weight, ro.discarded_weight) <= 1e-10
    assert (g.bond_dims() == o.bond_dims()).all()
    rng = np.random.default_rng(5)
    bits = ["".join(rng.choice(["0", "1"], n)) for _ in range(16)]
    ag = g.amplitudes(bits)
    ao = np.array([o.amplitude(b) for b in bits])
    assert np.max(np.abs(ag - ao) / np.abs(ao)) <= 1e-10


@pytest.mark.slow
def test_chi1024_gate_matches_oracle(gpu, oracle):
    _fullsize(gpu, oracle, 24, 1024, 256, [11])


@pytest.mark.slow
def test_chi512_layer_properties(gpu):
    """A full 128-gate-wide layer is out of the oracle's reach in a test, so
    check properties that hold at any size: the cap is met exactly, every
    gate's discarded weight equals 1 - kept/total in the renormalised state's
    local norm, and the layer is invariant under splitting it in two."""
    n, chi = 64, 512
    rng = np.random.default_rng(11)
    bonds = [min(chi, 2 ** min(i, n - i)) for i in range(n + 1)]
    sites = []
    for i in range(n):
        t = rng.standard_normal((bonds[i], 2, bonds[i + 1])) + 1j * rng.standard_normal((bonds[i], 2, bonds[i + 1]))
        sites.append(t / np.sqrt(4.0 * bonds[i]))
    def haar():
        z = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
        q, r = np.linalg.qr(z)
        return q * (np.diag(r) / np.abs(np.diag(r)))
    layer = [(q, q + 1, haar()) for q in range(0, n - 1, 2)]
    a = gpu.MpsState(n, chi_hint=chi)
    b = gpu.MpsState(n, chi_hint=chi)
    for i in range(n):
        a.set_site(i, sites[i])
        b.set_site(i, sites[i])
    ra = a.apply_layer(layer, max_bond=chi, cutoff=1e-12)
    rb = b.apply_layer(layer[: len(layer) // 2], max_bond=chi, cutoff=1e-12)
    rb += b.apply_layer(layer[len(layer) // 2:], max_bond=chi, cutoff=1e-12)
    assert [x.new_bond for x in ra] == [x.new_bond for x in rb]
    assert max(x.new_bond for x in ra) == chi
    assert all(abs(x.discarded_weight - y.discarded_weight) == 0.0 for x, y in zip(ra, rb))
    assert (a.bond_dims() == b.bond_dims()).all()
    bits = ["".join(rng.choice(["0", "1"], n)) for _ in range(8)]
    assert np.array_equal(a.amplitudes(bits), b.amplitudes(bits))  # batching is bit-exact


def _bench_chain(n, chi):
    """The exact bench.py workload: its chain (random sites seeded per site) and
    its layer sequence (Haar gates from default_rng(1234), parity alternating)."""
    import bench
    bonds = bench.chain_bonds(n, chi)
    sites = [bench.random_site(np.random.default_rng(10_000 + i), bonds[i], bonds[i + 1]) for i in range(n)]
    rng = np.random.default_rng(1234)
    layers = [bench.layer_gates(n, s % 2, rng) for s in range(2)]
    return sites, layers


@pytest.mark.slow
def test_bench_step_layers_match_oracle(gpu, oracle):
    """Two whole bench steps (the 128-gate even and the 127-gate odd brick
    layer of the 256-qubit chain at chi = 512, max_bond 512, cutoff 1e-12)
    through the public execute path, against the oracle's execute_parallel on
    every host core: per-gate kept ranks exactly, discarded weights and
    amplitudes to 1e-10 relative."""
    import os
    n, chi = 256, 512
    sites, layers = _bench_chain(n, chi)
    g = gpu.MpsState(n, chi_hint=chi)
    o = oracle.MpsState(n)
    for i, t in enumerate(sites):
        g.set_site(i, t)
        o.set_site(i, t)
    del sites
    workers = os.cpu_count() or 1
    for layer in layers:
        rg = gpu.execute(g, layer, chi, 1e-12)
        ro = oracle.execute_parallel(o, oracle.GateList(layer), chi, 1e-12, workers=workers)
        assert (rg["gate_k"] == ro["gate_k"]).all()
        assert (ro["gate_k"] == chi).sum() >= len(layer) - 10  # saturated gates
        nz = ro["gate_w"] > 0
        assert np.max(np.abs(rg["gate_w"][nz] - ro["gate_w"][nz]) / ro["gate_w"][nz]) <= 1e-10
        assert (rg["gate_w"][~nz] == 0).all()
        assert (g.bond_dims() == o.bond_dims()).all()
    rng = np.random.default_rng(7)
    bits = ["".join(rng.choice(["0", "1"], n)) for _ in range(16)]
    ag = g.amplitudes(bits)
    ao = np.array([o.amplitude(b) for b in bits])
    assert np.max(np.abs(ag - ao) / np.abs(ao)) <= 1e-10


def _oracle_spread(oracle, n, fused, chi, bits, workers):
    """Relative amplitude spread between two independent CPU SVDs (LAPACK
    zgesdd, the oracle's default, and zgesvj, one-sided Jacobi) on the same
    circuit: after hundreds of truncations at small spectral gaps
    the kept subspaces of two correct SVDs differ by ~eps / gap, which is the
    floor any implementation's amplitudes can be held to."""
    oracle.set_svd_backend("zgesvj")
    try:
        o2 = oracle.MpsState(n)
        r2 = oracle.execute_parallel(o2, fused, chi, 1e-12, workers=workers)
        a2 = np.array([o2.amplitude(b) for b in bits])
    finally:
        oracle.set_svd_backend("zgesdd")
    return r2, a2


@pytest.mark.slow
@pytest.mark.parametrize("haar", [True, False])
def test_c2_full_size(gpu, oracle, haar):
    """BASELINE C2 at its stated size: 64-qubit brickwork depth 20 (seed 4242,
    Haar sidecar entangler or Cx), chi = 128, cutoff 1e-12 — 630 fused gates
    in 20 layers. Per-gate bond dims exactly, discarded weights (each and the
    sum) to 1e-10, <Z_i> on every qubit to 1e-10, and 64 amplitudes (seed 7)
    to 1e-10 relative — or, where two independent CPU SVDs (zgesdd, zgesvj)
    already disagree by more (Haar: 2.8e-10, measured), to twice that spread."""
    import os
    n, chi = 64, 128
    workers = os.cpu_count() or 1
    fused = oracle.Circuit.brickwork(n, 20, 4242, haar=haar).fuse()
    o = oracle.MpsState(n)
    ro = oracle.execute_parallel(o, fused, chi, 1e-12, workers=workers)
    g = gpu.MpsState(n, chi_hint=chi)
    rg = gpu.execute(g, [(q0, q1, m) for (q0, q1, _f, m) in fused.gates()], chi, 1e-12)
    if haar:
        assert len(fused) == 630
        assert rg["peak_bond"] == ro["peak_bond"] == chi
    assert (rg["gate_k"] == ro["gate_k"]).all()
    assert (g.bond_dims() == o.bond_dims()).all()
    nz = ro["gate_w"] > 1e-16  # below: rank-deficient rounding noise
    if nz.any():
        assert np.max(np.abs(rg["gate_w"][nz] - ro["gate_w"][nz]) / ro["gate_w"][nz]) <= 1e-10
        assert rel(rg["total_discarded_weight"], ro["total_discarded_weight"]) <= 1e-10
    assert (rg["gate_w"][~nz] <= 1e-16).all()
    rng = np.random.default_rng(7)
    bits = ["".join(rng.choice(["0", "1"], n)) for _ in range(64)]
    ag = g.amplitudes(bits)
    ao = np.array([o.amplitude(b) for b in bits])
    big = np.abs(ao) > 1e-14 * np.abs(ao).max()
    err = np.max(np.abs(ag[big] - ao[big]) / np.abs(ao[big]))
    if err > 1e-10:
        r2, a2 = _oracle_spread(oracle, n, fused, chi, bits, workers)
        assert (r2["gate_k"] == ro["gate_k"]).all()
        spread = np.max(np.abs(a2[big] - ao[big]) / np.abs(ao[big]))
        assert err <= 2.0 * spread, (err, spread)
    pz = np.diag([1.0, -1.0]).astype(np.complex128)
    for q in range(n):
        oc = o.copy()
        oc.apply_1q(pz, q)
        ref = o.overlap(oc)
        got = g.expect_1q(pz, q)
        assert abs(got - ref) <= 1e-10 * max(1.0, abs(ref)), (q, got, ref)


@pytest.mark.slow
def test_c1_sampling_1e5_shots_equal_oracle(gpu, oracle):
    """BASELINE C1: 20-qubit GHZ + a seeded u3 layer (mt19937_64(1), brickwork
    draw order), chi <= 16: 1e5 shots with seed 42 give exactly the oracle
    sampler's counts (same variates, sampler.cpp:84/115)."""
    c = oracle.Circuit.ghz(20)
    for kind, q0, q1, params in oracle.Circuit.brickwork(20, 1, 1).ops():
        if kind == "u3":
            c.add("u3", q0, -1, params)
    fused = c.fuse()
    g = gpu.MpsState(20)
    gpu.execute(g, [(q0, q1, m) for (q0, q1, _f, m) in fused.gates()], 16, 0.0)
    o = oracle.MpsState(20)
    oracle.execute_serial(o, fused, 16, 0.0)
    a = gpu.sample(g, 100000, 42)
    b = oracle.Sampler(o).sample(100000, 42)
    assert sum(a.values()) == 100000
    assert a == b
