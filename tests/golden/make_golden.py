"""Writes the committed oracle fixtures for the BASELINE configs that are too
large to run through the CPU oracle inside a GPU test (TEST INFRASTRUCTURE).

  python tests/golden/make_golden.py c3   # tests/golden/c3_full.npz
  python tests/golden/make_golden.py c4   # tests/golden/c4_window.npz

c3: BASELINE C3 at its stated size — 100-qubit random brickwork of depth 32
    with non-adjacent CX gates (every 4th pair of an entangling layer becomes
    cx q[p], q[p+d], d = 2 + (draw % 3)), SWAP-routed by decompose_nonlocal
    (fusion.cpp:137-161), chi = 512, cutoff 1e-12.
c4: a BASELINE C4 window — disordered non-Clifford TFIM Trotter steps
    (cx; rz(-2 J dt); cx on even then odd bonds, rx(-2 h_i dt) on every site;
    J dt = 0.8, h_i dt = 0.8 + 0.2 (u_i - 1/2), u_i from mt19937_64(256)) on
    24 qubits until the centre bond reaches chi = 1024, plus two steps.

Each fixture holds the local gate list (the GPU test feeds it to the public
execute path as is), the oracle's per-gate kept rank and discarded weight in
gate order (SWAPs included), the final bond dims, 64 amplitudes of seeded
random bit strings, and <Z_q>, <X_q> (P9 definition, overlap(psi, O_q psi)).
The oracle run uses LAPACK zgesdd (Eigen BDCSVD's divide-and-conquer family);
the same circuit is re-run with a second SVD (c4: LAPACK zgesvj, one-sided
Jacobi; c3: zgesvd, bidiagonal QR iteration, zgesvj being too slow for ~2000
1024 x 1024 thetas on 8 cores) and the fixture records that both give the
same kept ranks and discarded weights within 1e-10, plus the amplitude spread
between the two runs. For c3, sampled saturated thetas of the run itself also
go through zgesvj (kept rank, weight). This is the oracle's own pin, since the
reference cannot be built here (Eigen3 absent).
"""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from tests.helpers import MT19937_64  # noqa: E402

PZ = np.diag([1.0, -1.0]).astype(np.complex128)
PX = np.array([[0, 1], [1, 0]], dtype=np.complex128)


def haar(rng):
    z = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def c3_circuit(n=100, depth=32, seed=2601):
    c = O.Circuit(n)
    rng = np.random.default_rng(seed)
    for layer in range(depth):
        for i, p in enumerate(range(layer % 2, n - 1, 2)):
            if i % 4 == 3:
                d = 2 + int(rng.integers(3))
                if p + d < n:
                    c.add("cx", p, p + d)
                    continue
            c.add("u4", p, p + 1, matrix=haar(rng))
    return c.fuse().decompose_nonlocal(n)


def tfim_step(n, u, jdt=0.8):
    c = O.Circuit(n)
    for parity in (0, 1):
        for p in range(parity, n - 1, 2):
            c.add("cx", p, p + 1)
            c.add("rz", p + 1, -1, (-2 * jdt,))
            c.add("cx", p, p + 1)
    for q in range(n):
        c.add("rx", q, -1, (-2 * (0.8 + 0.2 * (u[q] - 0.5)),))
    return c.fuse()


def run_oracle(n, gate_list, chi, cutoff, workers, pin=None):
    """execute_parallel layer by layer over the (local) list (the same layer
    plan the one-call run uses); reports back in gate order. pin(o, layer,
    gates) runs before each layer (the SVD pin samples its thetas)."""
    o = O.MpsState(n)
    layer_of, nl = gate_list.layer_of()
    gates = gate_list.gates()
    k = np.empty(len(gates), dtype=np.int64)
    w = np.empty(len(gates))
    for L in range(nl):
        idx = np.nonzero(layer_of == L)[0]
        lg = [(gates[i][0], gates[i][1], gates[i][3]) for i in idx]
        if pin is not None:
            pin(o, L, lg)
        r = O.execute_parallel(o, O.GateList(lg), chi, cutoff, workers=workers)
        k[idx] = r["gate_k"]
        w[idx] = r["gate_w"]
    return o, k, w


def theta_of(o, q, u):
    """apply_2q_local's theta (gate_apply.cpp:121-131): (2 Dl) x (2 Dr)."""
    a, b = o.site(q), o.site(q + 1)
    m = np.einsum("lam,mbr->labr", a, b)
    dl, dr = a.shape[0], b.shape[2]
    t = np.einsum("xy,lyr->lxr", u, m.reshape(dl, 4, dr)).reshape(dl, 2, 2, dr)
    return t.reshape(2 * dl, 2 * dr)


def make_pin(chi, cutoff, every, per_layer, start, workers, log):
    """Pin the oracle's SVD decisions on the fixture's own matrices: sampled
    saturated thetas go through zgesdd and zgesvj (one-sided Jacobi, an
    unrelated algorithm); kept ranks must agree and discarded weights to 1e-10."""
    from concurrent.futures import ThreadPoolExecutor

    def pin(o, L, lg):
        if L < start or (L - start) % every:
            return
        bonds = o.bond_dims()
        cand = [(q0, u) for q0, q1, u in lg if q1 >= 0 and bonds[q0] == bonds[q0 + 1] == bonds[q0 + 2] == chi]
        for q0, u in cand[:per_layer]:
            th = theta_of(o, q0, u)
            res = {}
            for name in ("zgesdd", "zgesvj"):
                O.set_svd_backend(name)
                _, s_, _, w_ = O.svd(th, chi, cutoff)
                res[name] = (len(s_), w_)
            O.set_svd_backend("zgesdd")
            (k1, w1), (k2, w2) = res["zgesdd"], res["zgesvj"]
            log.append({"layer": int(L), "q": int(q0), "k_zgesdd": k1, "k_zgesvj": k2, "w_zgesdd": w1,
                        "w_zgesvj": w2, "w_rel_diff": abs(w1 - w2) / max(w1, 1e-300)})
            print(f"  pin layer {L} gate {q0}: k {k1} / {k2}, w {w1:.3e} / {w2:.3e}, rel diff "
                  f"{log[-1]['w_rel_diff']:.2e}", flush=True)
    return pin


def observables(o, n, qs, workers, seed=7, count=64):
    rng = np.random.default_rng(seed)
    bits = ["".join(rng.choice(["0", "1"], n)) for _ in range(count)]
    amps = np.array([o.amplitude(b) for b in bits])

    def ex(args):
        op, q = args
        oc = o.copy()
        oc.apply_1q(op, q)
        return o.overlap(oc)

    with ThreadPoolExecutor(workers) as pool:  # ctypes releases the GIL
        z = np.array(list(pool.map(ex, [(PZ, q) for q in qs])))
        x = np.array(list(pool.map(ex, [(PX, q) for q in qs])))
    return bits, amps, z, x


def save(name, n, chi, cutoff, gates, k, w, bonds, bits, amps, qs, z, x, meta):
    q0 = np.array([g[0] for g in gates], dtype=np.int32)
    q1 = np.array([g[1] for g in gates], dtype=np.int32)
    mats = np.zeros((len(gates), 4, 4), dtype=np.complex128)
    for i, g in enumerate(gates):
        m = g[3]
        mats[i, : m.shape[0], : m.shape[1]] = m
    np.savez_compressed(os.path.join(HERE, name + ".npz"), n=n, chi=chi, cutoff=cutoff, q0=q0, q1=q1, mats=mats,
                        k=k, w=w, bonds=bonds, bits=np.array(bits), amps=amps, qs=np.array(qs), z=z, x=x)
    with open(os.path.join(HERE, name + ".json"), "w") as f:
        json.dump(meta, f, indent=1)


def make(which, workers):
    t0 = time.time()
    cutoff = 1e-12
    if which == "c3":
        n, chi = 100, 512
        gl = c3_circuit()
        qs = list(range(0, n, 4))
        meta = {"config": "C3: 100-qubit Haar brickwork depth 32, every 4th pair a non-adjacent cx (d = 2..4), "
                          "SWAP-routed, chi=512, cutoff 1e-12, numpy default_rng(2601)"}
    else:
        n, chi = 24, 1024
        e = MT19937_64(256)
        u = [e.unit() for _ in range(n)]
        o = O.MpsState(n)
        gates_all, steps = [], 0
        extra = None
        while extra is None or extra > 0:
            step = tfim_step(n, u)
            O.execute_parallel(o, step, chi, cutoff, workers=workers)
            gates_all.extend(step.gates())
            steps += 1
            if extra is not None:
                extra -= 1
            elif o.bond_dims().max() >= chi:
                extra = 2
            print(f"c4 step {steps}: max bond {o.bond_dims().max()}", flush=True)
        gl = O.GateList([(q0, q1, m) for (q0, q1, _f, m) in gates_all])
        qs = list(range(n))
        meta = {"config": f"C4 window: 24-qubit disordered TFIM (J dt 0.8, h_i dt 0.8+0.2(u_i-1/2), "
                          f"u_i from mt19937_64(256)), {steps} Trotter steps (centre bond reaches 1024, then 2 "
                          f"more), chi=1024, cutoff 1e-12", "steps": steps}
    gates = gl.gates()
    second = "zgesvj" if which == "c4" else "zgesvd"
    print(f"{which}: {len(gates)} local gates, running the oracle (zgesdd) on {workers} workers", flush=True)
    O.set_svd_backend("zgesdd")
    pins = []
    pin = make_pin(chi, cutoff, every=4, per_layer=2, start=16, workers=workers, log=pins) if which == "c3" else None
    o, k, w = run_oracle(n, gl, chi, cutoff, workers, pin)
    t1 = time.time()
    print(f"{which}: zgesdd run {t1 - t0:.0f} s, peak bond {k.max()}", flush=True)
    bonds = o.bond_dims()
    bits, amps, z, x = observables(o, n, qs, workers)
    print(f"{which}: observables {time.time() - t1:.0f} s", flush=True)
    del o
    # the same circuit through a second SVD: kept ranks, weights, and the
    # amplitude spread two correct SVDs leave after many truncations (P10)
    O.set_svd_backend(second)
    t2 = time.time()
    o2, k2, w2 = run_oracle(n, gl, chi, cutoff, workers)
    O.set_svd_backend("zgesdd")
    nz = w > 1e-16
    w_rel = float(np.max(np.abs(w2[nz] - w[nz]) / w[nz])) if nz.any() else 0.0
    amps2 = np.array([o2.amplitude(b) for b in bits])
    a_rel = float(np.max(np.abs(amps2 - amps) / np.abs(amps)))
    meta.update({
        "n": n, "chi": chi, "cutoff": cutoff, "local_gates": len(gates),
        "saturated_gates": int((k == chi).sum()), "peak_bond": int(k.max()),
        "total_discarded_weight": float(w.sum()),
        "second_svd": second,
        "zgesvj_check": {"second_svd": second, "kept_ranks_equal": bool((k2 == k).all()),
                         "rank_mismatches": int((k2 != k).sum()),
                         "max_rel_w_diff": w_rel, "max_rel_amp_diff": a_rel,
                         "bonds_equal": bool((o2.bond_dims() == bonds).all()), "seconds": time.time() - t2},
        "svd_pins": pins,
        "oracle_seconds": t1 - t0, "workers": workers,
        "generator": "tests/golden/make_golden.py " + which,
    })
    if pins:
        # weights at the rounding level (a SWAP undoing an earlier SWAP leaves a
        # theta of rank <= chi: w ~ 1e-30, two SVDs' noise) carry no information
        real = [p for p in pins if p["w_zgesdd"] > 1e-10]
        meta["svd_pin_summary"] = {"samples": len(pins), "samples_with_w_above_1e-10": len(real),
                                   "kept_ranks_equal": all(p["k_zgesdd"] == p["k_zgesvj"] for p in pins),
                                   "max_w_rel_diff_w_above_1e-10": max((p["w_rel_diff"] for p in real), default=0.0)}
    print(json.dumps(meta, indent=1), flush=True)
    save({"c3": "c3_full", "c4": "c4_window"}[which], n, chi, cutoff, gates, k, w, bonds, bits, amps, qs, z, x,
         meta)


if __name__ == "__main__":
    make(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else (os.cpu_count() or 1))
