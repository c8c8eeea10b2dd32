import sys; sys.path.insert(0, '.')
import numpy as np
from oracle import oracle as O
import paper_2601_04422_b200 as P
from tests.helpers import CX, HAD, SWAP
g = P.MpsState(4); o = O.MpsState(4)
g.apply_1q(HAD, 0); o.apply_1q(HAD, 0)
for (u, q) in [(SWAP, 0), (SWAP, 1), (CX, 2), (SWAP, 1), (SWAP, 0)]:
    rg = g.apply_2q_local(u, q); ro = o.apply_2q_local(u, q)
    print(q, rg, ro, g.bond_dims(), o.bond_dims(), "norm", g.norm(), o.norm())
    for i in range(4):
        a, b = g.site(i), o.site(i)
        print("   site", i, a.shape, np.round(a.reshape(-1), 3), b.shape, np.round(b.reshape(-1), 3))
