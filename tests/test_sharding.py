"""Host logic of the site-sharded chain on CPU: the library's
shard bounds and layer partitioning (mpsim_shard_bounds /
mpsim_shard_partition_layer, csrc/shard.cu), the straddle handshake between
neighbouring ranks, and the whole exchange protocol with real site bytes,
checked with world_size-2 gloo process groups and the CPU oracle as compute."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_04422_b200.sharded import partition_layer, shard_bounds


def _layer(n, parity):
    return [(q, q + 1, np.eye(4)) for q in range(parity, n - 1, 2)]


@pytest.mark.parametrize("n,world", [(16, 2), (256, 8), (100, 4), (10, 3)])
def test_bounds_even_and_covering(n, world):
    b = shard_bounds(n, world)
    assert b[0] == 0 and b[-1] == n and len(b) == world + 1
    assert all(x % 2 == 0 for x in b[:-1])
    assert all(b[i + 1] - b[i] >= 2 for i in range(world))


@pytest.mark.parametrize("n,world,chi", [(256, 4, 512), (256, 8, 512), (64, 4, 128), (20, 2, 16)])
def test_cost_weighted_bounds_balance(n, world, chi):
    b = shard_bounds(n, world, chi)
    assert b[0] == 0 and b[-1] == n and all(x % 2 == 0 for x in b[:-1])
    assert all(b[i + 1] - b[i] >= 2 for i in range(world))
    bond = [min(chi, 2 ** min(q, n - q)) for q in range(n + 1)]
    cost = [bond[q] * bond[q + 1] * bond[min(q + 2, n)] for q in range(n)]
    shard = [sum(cost[b[r]:b[r + 1]]) for r in range(world)]
    even = shard_bounds(n, world)
    shard_even = [sum(cost[even[r]:even[r + 1]]) for r in range(world)]
    # never worse than the even split, within ~12 % of perfect balance
    assert max(shard) <= max(shard_even) + 1e-9
    assert max(shard) <= 1.12 * sum(cost) / world


@pytest.mark.parametrize("n,world", [(16, 2), (64, 4), (256, 8)])
def test_every_gate_applied_once(n, world):
    b = shard_bounds(n, world, 512 if n >= 64 else None)
    for parity in (0, 1):
        gates = _layer(n, parity)
        seen = []
        flags = []
        for r in range(world):
            local, sl, sr = partition_layer(gates, b[r], b[r + 1], r, world)
            seen += [q0 + b[r] for q0, _, _ in local]
            flags.append((sl, sr))
        assert sorted(seen) == [g[0] for g in gates]
        # even layers never straddle (boundaries are even); odd layers straddle at each boundary
        for r in range(world - 1):
            assert flags[r][1] == flags[r + 1][0] == (parity == 1)


def test_nonlocal_rejected():
    with pytest.raises(ValueError):
        partition_layer([(0, 2, np.eye(4))], 0, 4, 0, 1)


def _worker(rank, world, port, n, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = shard_bounds(n, world)
    ok = True
    for parity in (0, 1):
        local, sl, sr = partition_layer(_layer(n, parity), b[rank], b[rank + 1], rank, world)
        flags = [None] * world
        dist.all_gather_object(flags, (sl, sr, len(local)))
        for r in range(world - 1):
            ok &= flags[r][1] == flags[r + 1][0]
        ok &= sum(f[2] for f in flags) == len(_layer(n, parity))
    out[rank] = ok
    dist.destroy_process_group()


def test_gloo_two_ranks_handshake():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, 20, out)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    assert all(p.exitcode == 0 for p in ps)
    assert out[0] and out[1]


def _protocol_worker(rank, world, port, out):
    """The exchange protocol of csrc/shard.cu with real site tensors: each rank
    holds an oracle chain of its sites + a ghost slot; per layer it partitions
    with the library's planner, lends / borrows the boundary site (extents,
    then bytes, over gloo), applies its gates, and returns the updated ghost.
    The gathered chain must equal a one-process run bit for bit."""
    import torch
    from oracle import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, chi, layers = 14, 8, 6
    full = O.MpsState.random(n, chi, 4242)
    b = shard_bounds(n, world, chi)
    lo, hi = b[rank], b[rank + 1]
    k = hi - lo
    ghost = k if rank < world - 1 else None
    st = O.MpsState(k + (1 if ghost is not None else 0))
    for i in range(lo, hi):
        st.set_site(i - lo, full.site(i))

    def send(t, dst):
        dist.send(torch.tensor(list(t.shape), dtype=torch.int64), dst)
        dist.send(torch.from_numpy(np.ascontiguousarray(t)), dst)

    def recv(src):
        shp = torch.zeros(3, dtype=torch.int64)
        dist.recv(shp, src)
        t = torch.zeros(tuple(int(x) for x in shp), dtype=torch.complex128)
        dist.recv(t, src)
        return t.numpy()

    rng = np.random.default_rng(99)
    plan = []
    for L in range(layers):
        plan.append([(q, q + 1, O.haar_unitary(4, int(rng.integers(1 << 30)))) for q in range(L % 2, n - 1, 2)])
    for layer in plan:
        local, sl, sr = partition_layer(layer, lo, hi, rank, world)
        # exchange in: rank r+1's first site -> rank r's ghost (rank parity
        # orders the blocking gloo calls)
        for phase in (0, 1):
            if sl and rank % 2 == phase:
                send(st.site(0), rank - 1)
            if sr and rank % 2 != phase:
                st.set_site(ghost, recv(rank + 1))
        for q0, q1, u in local:
            st.apply_2q_local(u, min(q0, q1), max_bond=chi, cutoff=1e-12)
        # exchange out: the updated ghost goes back as rank r+1's first site
        for phase in (0, 1):
            if sr and rank % 2 == phase:
                send(st.site(ghost), rank + 1)
            if sl and rank % 2 != phase:
                st.set_site(0, recv(rank - 1))
    mine = {i: st.site(i - lo) for i in range(lo, hi)}
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    if rank == 0:
        ref = O.MpsState.random(n, chi, 4242)
        for layer in plan:
            for q0, q1, u in layer:
                ref.apply_2q_local(u, q0, max_bond=chi, cutoff=1e-12)
        got = {}
        for p in parts:
            got.update(p)
        out["ok"] = all(np.array_equal(got[i], ref.site(i)) for i in range(n))
        out["bonds"] = [got[i].shape[0] for i in range(n)] == list(ref.bond_dims()[:-1])
    dist.destroy_process_group()


def test_gloo_two_ranks_exchange_protocol_moves_sites():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    ps = [ctx.Process(target=_protocol_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
    assert all(p.exitcode == 0 for p in ps)
    assert out["ok"] and out["bonds"]


def test_partition_layer_roundtrips_matrices():
    u = np.arange(16, dtype=np.complex128).reshape(4, 4) * (1 + 0.5j)
    v = np.array([[0, 1j], [1, 0]])
    local, sl, sr = partition_layer([(5, 6, u), (3, -1, np.eye(2)), (6, -1, v), (7, 8, u)], 4, 8, 1, 3)
    assert not sl and sr  # (7, 8) straddles into the ghost slot 4
    assert [(q0, q1) for q0, q1, _ in local] == [(1, 2), (2, -1), (3, 4)]
    assert np.array_equal(local[0][2], u) and np.array_equal(local[1][2], v)
