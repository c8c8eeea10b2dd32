"""Multi-GPU parity of the library's shard layer (csrc/shard.cu): a site-sharded
chain (NCCL boundary exchange) must give the same kept ranks, sites and
amplitudes as the same work on one GPU — brick layers, a circuit with
non-local gates whose SWAP chains cross shard boundaries, sharded queries,
centre moves, and perfect sampling. No torch: the NCCL id is bootstrapped
over a socket, sites are compared through files.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/mgpu_check.py
"""
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_04422_b200 as P  # noqa: E402
from paper_2601_04422_b200 import sharded  # noqa: E402


def haar4(rng):
    z = (rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))) / np.sqrt(2)
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def nonlocal_circuit(n, depth, seed):
    rng = np.random.default_rng(seed)
    cx = np.eye(4, dtype=complex)[[0, 1, 3, 2]]
    gates = []
    for layer in range(depth):
        for i, p in enumerate(range(layer % 2, n - 1, 2)):
            d = 2 + int(rng.integers(3))
            if i % 4 == 3 and p + d < n:
                gates.append((p, p + d, cx))
            else:
                gates.append((p, p + 1, haar4(rng)))
    return gates


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    tmp = os.environ.get("MGPU_TMP", os.path.join(tempfile.gettempdir(), "mgpu_check"))
    os.makedirs(tmp, exist_ok=True)
    n, chi, layers = int(os.environ.get("NQ", "40")), int(os.environ.get("CHI", "64")), 6
    bonds = [min(chi, 2 ** min(i, n - i)) for i in range(n + 1)]
    sites = []
    for i in range(n):
        r = np.random.default_rng(500 + i)
        t = r.standard_normal((bonds[i], 2, bonds[i + 1])) + 1j * r.standard_normal((bonds[i], 2, bonds[i + 1]))
        sites.append(t / np.sqrt(4.0 * bonds[i]))
    rng = np.random.default_rng(77)
    plan = [[(q, q + 1, haar4(rng)) for q in range(L % 2, n - 1, 2)] for L in range(layers)]

    chain = sharded.ShardedChain(n, chi, rank, world, device=local)
    for i in range(chain.lo, chain.hi):
        chain.set_site(i, sites[i])
    for layer in plan:
        chain.apply_layer(layer, chi, 1e-12)
    brng = np.random.default_rng(9)
    qbits = ["".join(brng.choice(["0", "1"], n)) for _ in range(64)]
    s_amp = chain.amplitudes(qbits)
    s_norm = chain.norm()
    pz = np.diag([1.0, -1.0]).astype(np.complex128)
    qs = [0, n // 3, n // 2, n - 1]
    s_exp = [chain.expect_1q(pz, q) for q in qs]
    np.savez(os.path.join(tmp, f"a{rank}.npz"), **{str(i): chain.site(i) for i in range(chain.lo, chain.hi)})
    cc = (2 * n) // 3
    chain.move_center(cc)
    np.savez(os.path.join(tmp, f"b{rank}.npz"), **{str(i): chain.site(i) for i in range(chain.lo, chain.hi)})
    nrm = chain.norm()
    if chain.lo <= cc < chain.hi:
        chain.set_site(cc, chain.site(cc) / nrm)
    chain.sample(3000, 5, chunk=1024)  # warm-up
    chain.barrier()
    t0 = time.perf_counter()
    s_counts = chain.sample(3000, 5, chunk=1024)
    t_sample = chain.max_over_ranks(time.perf_counter() - t0)
    # a circuit with non-local CX gates: SWAP chains cross the shard boundaries
    gates = nonlocal_circuit(n, 10, 2601)
    ch2 = sharded.ShardedChain(n, chi, rank, world, device=local)
    st2 = ch2.execute(gates, chi, 1e-12)
    b2 = ch2.bond_dims()
    np.save(os.path.join(tmp, f"c{rank}.npy"), b2)
    c_amp = ch2.amplitudes(qbits)
    chain.barrier()
    if rank == 0:
        def gather(tag):
            full = {}
            for r in range(world):
                with np.load(os.path.join(tmp, f"{tag}{r}.npz")) as f:
                    full.update({int(k): f[k] for k in f.files})
            return full
        full = gather("a")
        ref = P.MpsState(n, chi_hint=chi, device=local)
        for i in range(n):
            ref.set_site(i, sites[i])
        for layer in plan:
            ref.apply_layer(layer, chi, 1e-12)
        site_eq = all(np.array_equal(full[i], ref.site(i)) for i in range(n))
        b = ref.amplitudes(qbits)
        q_amp = float(np.max(np.abs(s_amp - b) / np.abs(b)))
        q_norm = abs(s_norm - ref.norm()) / ref.norm()
        q_exp = max(abs(e - ref.expect_1q(pz, q)) for e, q in zip(s_exp, qs))
        ok = site_eq and q_amp <= 1e-12 and q_norm <= 1e-12 and q_exp <= 1e-12
        print(f"MGPU world={world} n={n} chi={chi} layers: sites_bit_identical={site_eq} sharded queries: "
              f"amp {q_amp:.2e} norm {q_norm:.2e} <Z> {q_exp:.2e} {'OK' if ok else 'FAIL'}", flush=True)
        full2 = gather("b")
        ref.move_center(cc)
        site_eq2 = all(np.array_equal(full2[i], ref.site(i)) for i in range(n))
        ref.set_site(cc, ref.site(cc) / ref.norm())
        r_counts = P.sample(ref, 3000, 5)
        ok2 = site_eq2 and s_counts == r_counts
        print(f"MGPU world={world} move_center({cc}): sites_bit_identical={site_eq2}; sample(3000, seed 5): "
              f"{len(s_counts)} outcomes, {t_sample * 1e3:.1f} ms (max over ranks), "
              f"counts_equal={s_counts == r_counts} {'OK' if ok2 else 'FAIL'}", flush=True)
        ref2 = P.MpsState(n, chi_hint=chi, device=local)
        rs = P.execute(ref2, gates, chi, 1e-12)
        bounds = sharded.shard_bounds(n, world, chi)
        got_b = np.concatenate([np.load(os.path.join(tmp, f"c{r}.npy"))[:-1] for r in range(world)] + [[1]])
        a2 = ref2.amplitudes(qbits)
        c_err = float(np.max(np.abs(c_amp - a2)) / max(np.abs(a2).max(), 1e-300))
        print(f"  non-local circuit amplitudes: max |a| {np.abs(a2).max():.3e}, zeros {(a2 == 0).sum()}", flush=True)
        ok3 = bool((got_b == ref2.bond_dims()).all()) and c_err <= 1e-12 and st2["peak_bond"] == rs["peak_bond"] \
            and abs(st2["total_discarded_weight"] - rs["total_discarded_weight"]) <= 1e-12 * rs["total_discarded_weight"]
        print(f"MGPU world={world} non-local circuit ({len(gates)} gates, {st2['gates']} local, bounds {bounds}): "
              f"bonds_equal={bool((got_b == ref2.bond_dims()).all())} amp {c_err:.2e} peak {st2['peak_bond']} "
              f"w {st2['total_discarded_weight']:.6e} vs {rs['total_discarded_weight']:.6e} "
              f"{'OK' if ok3 else 'FAIL'}", flush=True)
        failed = not (ok and ok2 and ok3)
    else:
        failed = False
    chain.barrier()  # every rank leaves together (no rank left waiting on a failed one)
    if failed:
        sys.exit(1)


if __name__ == "__main__":
    main()
