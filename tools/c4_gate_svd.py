"""GPU SVD of the C4 window's truncating thetas (dumped by tools/c4_conditioning.py
DUMP=...) against numpy's LAPACK gesdd: kept rank, weight, and the distance
between the kept left subspaces, || U_k U_k^H - U'_k U'_k^H ||_2, and the
reconstruction error of the truncated product."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_04422_b200 as P  # noqa: E402

f = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c4_thetas.npz")
for i, (kk, ww) in enumerate(zip(f["k"], f["w"])):
    th = f[f"theta{i}"]
    u, s, vh, w = P.mps.svd(th, max_rank=1024, cutoff=1e-12)
    un, sn, vhn = np.linalg.svd(th, full_matrices=False)
    k = len(s)
    pg = u[:, :k] @ u[:, :k].conj().T
    pn = un[:, :k] @ un[:, :k].conj().T
    d = np.linalg.norm(pg - pn, 2)
    gap = (sn[k - 1] - sn[k]) / sn[k - 1] if k < len(sn) else 1.0
    rec_g = np.linalg.norm(u @ (s[:, None] * vh) - (un[:, :k] * sn[:k]) @ vhn[:k]) / np.linalg.norm(th)
    orth = np.linalg.norm(u.conj().T @ u - np.eye(k), 2)
    print(f"theta {i} {th.shape}: k {k} (ref {kk}), w {w:.6e} vs {ww:.6e} rel {abs(w - ww) / ww:.1e}; "
          f"||P_gpu - P_np|| {d:.2e}, rel gap at cut {gap:.2e}, ||U^H U - I|| {orth:.1e}, "
          f"truncated products differ {rec_g:.1e}", flush=True)
