import os, sys
import numpy as np
sys.path.insert(0, '.')
import oracle.oracle as O
import paper_2601_04422_b200 as P
from tests.helpers import gate_tuples
n, depth, chi = 24, 8, 32
c = O.Circuit(n)
rng = np.random.default_rng(2601)
for layer in range(depth):
    for i, p in enumerate(range(layer % 2, n - 1, 2)):
        if i % 4 == 3:
            d = 2 + int(rng.integers(3))
            if p + d < n:
                c.add("cx", p, p + d)
                continue
        z = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
        q, r = np.linalg.qr(z)
        c.add("u4", p, p + 1, matrix=q * (np.diag(r) / np.abs(np.diag(r))))
fused = c.fuse()
g = P.MpsState(n, chi_hint=chi)
try:
    rg = P.execute(g, gate_tuples(fused), chi, 1e-12)
    print("ok", rg["peak_bond"])
except Exception as e:
    print("FAIL", e)
