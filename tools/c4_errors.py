"""Prints the C4-window fixture errors of the GPU path (kept ranks, weights, amplitudes, <Z>, <X>)."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_04422_b200 as gpu
from tests.test_gpu_golden import _load, PZ, PX
name = sys.argv[1] if len(sys.argv) > 1 else "c4_window"
f, meta, gates = _load(name)
n, chi, cutoff = int(f["n"]), int(f["chi"]), float(f["cutoff"])
g = gpu.MpsState(n, chi_hint=chi)
rg = gpu.execute(g, gates, chi, cutoff)
k, w = f["k"], f["w"]
nz = w > 1e-16
print("k mismatches", int((rg["gate_k"] != k).sum()), "max rel w", float(np.max(np.abs(rg["gate_w"][nz] - w[nz]) / w[nz])))
ag = g.amplitudes([str(b) for b in f["bits"]]); ao = f["amps"]
rel = np.abs(ag - ao) / np.abs(ao)
print("amp rel err max %.3e median %.3e" % (rel.max(), np.median(rel)), "norm", g.norm() if hasattr(g, "norm") else "")
ez = max(abs(g.expect_1q(PZ, int(q)) - z) for q, z in zip(f["qs"], f["z"]))
ex = max(abs(g.expect_1q(PX, int(q)) - x) for q, x in zip(f["qs"], f["x"]))
print("max |<Z>| err %.3e, max |<X>| err %.3e" % (ez, ex))
trans = [1 if (2 * 1) else 0]
rw = np.where(nz, np.abs(rg["gate_w"] - w) / np.where(nz, w, 1), 0)
order = np.argsort(-rw)[:8]
print("worst w gates: idx, q0, q1, k, w_oracle, w_gpu, rel")
for i in order:
    print(int(i), int(f["q0"][i]), int(f["q1"][i]), int(k[i]), "%.6e %.6e %.2e" % (w[i], rg["gate_w"][i], rw[i]))
print("w>1e-16 gates:", int(nz.sum()), "of", len(w), " w range %.2e..%.2e" % (w[nz].min(), w[nz].max()))
