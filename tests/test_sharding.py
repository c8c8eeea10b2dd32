"""Host logic of the site-sharded chain on CPU: shard bounds,
layer partitioning, and the straddle handshake between neighbouring ranks,
checked with a world_size-2 gloo process group."""
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
