"""Multi-GPU parity: a site-sharded chain (NCCL boundary exchange) must give
the same kept ranks and amplitudes as the same layers on one GPU.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/mgpu_check.py
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_04422_b200 as P  # noqa: E402
from paper_2601_04422_b200 import sharded  # noqa: E402


def haar4(rng):
    z = (rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))) / np.sqrt(2)
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    n, chi, layers = int(os.environ.get("NQ", "40")), int(os.environ.get("CHI", "64")), 6
    bonds = [min(chi, 2 ** min(i, n - i)) for i in range(n + 1)]
    sites = []
    for i in range(n):
        r = np.random.default_rng(500 + i)
        t = r.standard_normal((bonds[i], 2, bonds[i + 1])) + 1j * r.standard_normal((bonds[i], 2, bonds[i + 1]))
        sites.append(t / np.sqrt(4.0 * bonds[i]))
    rng = np.random.default_rng(77)
    plan = [[(q, q + 1, haar4(rng)) for q in range(L % 2, n - 1, 2)] for L in range(layers)]

    chain = sharded.ShardedChain(n, chi, rank, world, device=local, dist=dist)
    for i in range(chain.lo, chain.hi):
        chain.set_site(i, sites[i])
    chain.finalize_setup()
    for layer in plan:
        chain.apply_layer(layer, chi, 1e-12)
    # sharded queries (environments passed rank to rank over NCCL)
    qbits = ["".join(np.random.default_rng(9).choice(["0", "1"], n)) for _ in range(64)]
    s_amp = chain.amplitudes(qbits)
    s_norm = chain.norm()
    pz = np.diag([1.0, -1.0]).astype(np.complex128)
    qs = [0, n // 3, n // 2, n - 1]
    s_exp = [chain.expect_1q(pz, q) for q in qs]
    mine = {i: chain.state.site(i - chain.lo) for i in range(chain.lo, chain.hi)}
    allsites = [None] * world
    dist.all_gather_object(allsites, mine)
    # centre move across the shards (QR sweeps handed rank to rank)
    cc = (2 * n) // 3
    chain.move_center(cc)
    mine2 = {i: chain.state.site(i - chain.lo) for i in range(chain.lo, chain.hi)}
    # normalise at the centre, then sample across the shards
    nrm = chain.norm()
    if chain.lo <= cc < chain.hi:
        chain.state.set_site(cc - chain.lo, chain.state.site(cc - chain.lo) / nrm)
    import time
    chain.sample(3000, 5, chunk=1024)  # warm-up (communicators, allocations)
    dist.barrier()
    t0 = time.perf_counter()
    s_counts = chain.sample(3000, 5, chunk=1024)
    t_sample = chain.max_over_ranks(time.perf_counter() - t0)
    allsites2 = [None] * world
    dist.all_gather_object(allsites2, mine2)
    if rank == 0:
        full = {}
        for d in allsites:
            full.update(d)
        ref = P.MpsState(n, chi_hint=chi, device=local)
        for i in range(n):
            ref.set_site(i, sites[i])
        for layer in plan:
            ref.apply_layer(layer, chi, 1e-12)
        rb = ref.bond_dims()
        got = P.MpsState(n, chi_hint=chi, device=local)
        for i in range(n):
            got.set_site(i, full[i])
        gb = got.bond_dims()
        bits = ["".join(np.random.default_rng(9).choice(["0", "1"], n)) for _ in range(64)]
        a, b = got.amplitudes(bits), ref.amplitudes(bits)
        err = float(np.max(np.abs(a - b) / np.abs(b)))
        q_amp = float(np.max(np.abs(s_amp - b) / np.abs(b)))
        q_norm = abs(s_norm - ref.norm()) / ref.norm()
        q_exp = max(abs(e - ref.expect_1q(pz, q)) for e, q in zip(s_exp, qs))
        ok = bool((gb == rb).all()) and err <= 1e-10 and q_amp <= 1e-10 and q_norm <= 1e-12 and q_exp <= 1e-10
        print(f"MGPU world={world} n={n} chi={chi} bonds_equal={bool((gb == rb).all())} "
              f"max_rel_amp_err={err:.2e} sharded_queries: amp {q_amp:.2e} norm {q_norm:.2e} "
              f"<Z> {q_exp:.2e} {'OK' if ok else 'FAIL'}", flush=True)
        full2 = {}
        for d in allsites2:
            full2.update(d)
        got2 = P.MpsState(n, chi_hint=chi, device=local)
        for i in range(n):
            got2.set_site(i, full2[i])
        ref.move_center(cc)
        mb_ok = bool((got2.bond_dims() == ref.bond_dims()).all())
        m_err = float(np.max(np.abs(got2.amplitudes(bits) - ref.amplitudes(bits)) / np.abs(ref.amplitudes(bits))))
        site_eq = all(np.array_equal(full2[i], ref.site(i)) for i in range(n))
        ref.set_site(cc, ref.site(cc) / ref.norm())
        r_counts = P.sample(ref, 3000, 5)
        ok3 = s_counts == r_counts
        print(f"MGPU world={world} n={n} chi={chi} sharded sample(3000, seed 5): {len(s_counts)} outcomes, "
              f"{t_sample * 1e3:.1f} ms (max over ranks), counts_equal={ok3} {'OK' if ok3 else 'FAIL'}", flush=True)
        ok2 = mb_ok and m_err <= 1e-10 and ok3
        print(f"MGPU world={world} n={n} chi={chi} move_center({cc}): bonds_equal={mb_ok} "
              f"max_rel_amp_err={m_err:.2e} sites_bit_identical={site_eq} {'OK' if ok2 else 'FAIL'}", flush=True)
        if not (ok and ok2):
            sys.exit(1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
