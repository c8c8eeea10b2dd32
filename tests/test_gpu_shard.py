"""The library's shard layer (csrc/shard.cu) at world size 1 on one GPU: the
same entry points the multi-GPU runs use (mpsim_gpu_shard_*), against the
single-state API. Multi-rank bit-identity (N = 2, 4) is checked by
tools/mgpu_check.py under torchrun (profiles/mgpu_parity_r02.txt)."""
import numpy as np
import pytest

from tests.helpers import CX

pytestmark = pytest.mark.gpu


def _haar(rng):
    z = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def test_shard_world1_matches_state(gpu, oracle):
    from paper_2601_04422_b200 import sharded
    n, chi = 16, 16
    o = oracle.MpsState.random(n, chi, 31)
    ch = sharded.ShardedChain(n, chi, 0, 1)
    ref = gpu.MpsState(n, chi_hint=chi)
    for i in range(n):
        ch.set_site(i, o.site(i))
        ref.set_site(i, o.site(i))
    rng = np.random.default_rng(3)
    for layer in range(4):
        gates = [(q, q + 1, _haar(rng)) for q in range(layer % 2, n - 1, 2)]
        st = ch.apply_layer(gates, 8, 1e-12)
        ref.apply_layer(gates, 8, 1e-12)
        assert st["device_ms"] > 0
    assert (ch.bond_dims() == ref.bond_dims()).all()
    assert all(np.array_equal(ch.site(i), ref.site(i)) for i in range(n))
    bits = ["".join(rng.choice(["0", "1"], n)) for _ in range(8)]
    assert np.array_equal(ch.amplitudes(bits), ref.amplitudes(bits))
    assert ch.norm() == ref.norm()
    pz = np.diag([1.0, -1.0]).astype(np.complex128)
    assert ch.expect_1q(pz, 5) == ref.expect_1q(pz, 5)
    ch.move_center(7)
    ref.move_center(7)
    assert ch.ortho_center == 7
    assert all(np.array_equal(ch.site(i), ref.site(i)) for i in range(n))
    # execute with non-local gates (SWAP-lowered and layered in the library)
    gl = [(0, 3, CX), (2, 9, CX), (5, 6, _haar(rng)), (12, 15, CX)]
    ch2 = sharded.ShardedChain(n, chi, 0, 1)
    r2 = gpu.MpsState(n, chi_hint=chi)
    s1 = ch2.execute(gl, chi, 1e-12)
    s2 = gpu.execute(r2, gl, chi, 1e-12)
    assert s1["gates"] == s2["gates"] and s1["peak_bond"] == s2["peak_bond"]
    assert (ch2.bond_dims() == r2.bond_dims()).all()
    assert np.array_equal(ch2.amplitudes(bits), r2.amplitudes(bits))


def test_shard_rejects_bad_arguments(gpu):
    from paper_2601_04422_b200 import sharded
    with pytest.raises(ValueError):
        sharded.ShardedChain(16, 16, 2, 2, nccl_id=b"\0" * 128)  # rank out of range
    ch = sharded.ShardedChain(8, 4, 0, 1)
    with pytest.raises(ValueError):
        ch.set_site(8, np.zeros((1, 2, 1)))
    with pytest.raises(ValueError):
        ch.apply_layer([(0, 2, CX)], 4, 0.0)  # layers must be local
