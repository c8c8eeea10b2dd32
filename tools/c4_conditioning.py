"""Conditioning of the C4-window fixture (TEST INFRASTRUCTURE / diagnostics):
re-runs the fixture's gate list with numpy's LAPACK SVD (gesdd), once as is
and once with every theta perturbed by a random relative 1e-16 before its SVD,
and prints how far the 64 fixture amplitudes move - the spread any correct
complex128 simulator must be allowed."""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
f = np.load(os.path.join(HERE, "..", "tests", "golden", "c4_window.npz"))
n, chi, cutoff = int(f["n"]), int(f["chi"]), float(f["cutoff"])


def run(eps, seed=3, dump=None):
    rng = np.random.default_rng(seed)
    sites = [np.zeros((1, 2, 1), complex) for _ in range(n)]
    for s in sites:
        s[0, 0, 0] = 1.0
    ks = []
    for q0, q1, m in zip(f["q0"], f["q1"], f["mats"]):
        q0, q1 = int(q0), int(q1)
        if q1 < 0:
            sites[q0] = np.einsum("ab,lbr->lar", m[:2, :2], sites[q0])
            continue
        a, b = sites[q0], sites[q0 + 1]
        dl, dr = a.shape[0], b.shape[2]
        t = np.einsum("lam,mbr->labr", a, b).reshape(dl, 4, dr)
        th = np.einsum("xy,lyr->lxr", m, t).reshape(2 * dl, 2 * dr)
        if eps:
            th = th * (1.0 + eps * (rng.standard_normal(th.shape) + 1j * rng.standard_normal(th.shape)))
        if not np.isfinite(th).all():
            raise RuntimeError(f"non-finite theta at gate ({q0}, {q1})")
        try:
            u, s, vh = np.linalg.svd(th, full_matrices=False)
        except np.linalg.LinAlgError:  # gesdd failure: the QR-iteration driver
            import scipy.linalg as sl
            u, s, vh = sl.svd(th, full_matrices=False, lapack_driver="gesvd")
        total = float((s * s).sum())
        keep = len(s)
        if total > 0:
            tail = 0.0
            while keep > 1 and tail + s[keep - 1] ** 2 <= cutoff * total:
                tail += s[keep - 1] ** 2
                keep -= 1
        else:
            keep = 1
        keep = min(keep, chi)
        w = float((s[keep:] ** 2).sum()) / total if total > 0 else 0.0
        sk = s[:keep] / np.sqrt(1.0 - w) if w > 0 else s[:keep]
        if dump is not None and w > 1e-16:
            dump.append((th.copy(), keep, w))
        sites[q0] = u[:, :keep].reshape(dl, 2, keep)
        sites[q0 + 1] = (sk[:, None] * vh[:keep]).reshape(keep, 2, dr)
        ks.append(keep)
    amps = []
    for bits in f["bits"]:
        env = np.ones((1,), complex)
        for i, c in enumerate(str(bits)):
            env = env @ sites[i][:, int(c), :]
        amps.append(env[0])
    return np.array(amps), np.array(ks)


t0 = time.time()
dumped = []
a0, k0 = run(0.0, dump=dumped)
if os.environ.get("DUMP"):
    np.savez_compressed(os.environ["DUMP"], **{f"theta{i}": d[0] for i, d in enumerate(dumped)},
                        k=np.array([d[1] for d in dumped]), w=np.array([d[2] for d in dumped]))
    print("dumped", len(dumped), "truncating thetas to", os.environ["DUMP"], flush=True)
    sys.exit(0)
print(f"numpy gesdd run {time.time() - t0:.0f} s; vs fixture (oracle zgesdd): max rel amp diff "
      f"{np.max(np.abs(a0 - f['amps']) / np.abs(f['amps'])):.2e}", flush=True)
for seed in (1, 2):
    a1, k1 = run(1e-16, seed)
    rel = np.abs(a1 - a0) / np.abs(a0)
    print(f"theta perturbed by 1e-16 (seed {seed}): kept ranks equal {bool((k1 == k0).all())}, "
          f"amplitudes max rel diff {rel.max():.2e}, median {np.median(rel):.2e}", flush=True)
