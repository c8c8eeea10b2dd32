"""Centre-move case for timing / ncu: a saturated random chain (n = 64, chi =
512 by default), left sweep to the last site then right sweep back to 0 (the
sampler's canonicalisation, sampler.cpp:46-47). Prints wall times."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_04422_b200 as P  # noqa: E402

n, chi = int(os.environ.get("NQ", "64")), int(os.environ.get("CHI", "512"))
bonds = [min(chi, 2 ** min(i, n - i)) for i in range(n + 1)]
g = P.MpsState(n, chi_hint=chi)
for i in range(n):
    r = np.random.default_rng(500 + i)
    a = r.standard_normal((bonds[i], 2, bonds[i + 1])) + 1j * r.standard_normal((bonds[i], 2, bonds[i + 1]))
    g.set_site(i, a / np.sqrt(4.0 * bonds[i]))
reps = int(os.environ.get("REPS", "2"))
for rep in range(reps):
    c = g.copy()
    c.synchronize()
    t0 = time.perf_counter()
    c.move_center(n - 1)
    c.synchronize()
    t1 = time.perf_counter()
    c.move_center(0)
    c.synchronize()
    t2 = time.perf_counter()
    print(f"rep {rep}: left sweep {1e3 * (t1 - t0):.1f} ms, right sweep {1e3 * (t2 - t1):.1f} ms, "
          f"bonds {list(c.bond_dims()[n // 2 - 2: n // 2 + 3])}", flush=True)
