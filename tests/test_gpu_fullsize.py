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
