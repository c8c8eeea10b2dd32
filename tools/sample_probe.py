"""Where the sampler's time goes on one GPU (n=64, chi=512 saturated random
chain): state copy, the two canonicalising QR sweeps, the site walk, and the
whole Sampler.sample. Wall times after one warm-up pass.

  python tools/sample_probe.py
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_04422_b200 as P  # noqa: E402
from paper_2601_04422_b200.mps import uniform_variates  # noqa: E402


def t(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) * 1e3


def main():
    n, chi = int(os.environ.get("NQ", "64")), int(os.environ.get("CHI", "512"))
    shots = int(os.environ.get("SHOTS", "3000"))
    bonds = [min(chi, 2 ** min(i, n - i)) for i in range(n + 1)]
    g = P.MpsState(n, chi_hint=chi)
    for i in range(n):
        r = np.random.default_rng(500 + i)
        a = r.standard_normal((bonds[i], 2, bonds[i + 1])) + 1j * r.standard_normal((bonds[i], 2, bonds[i + 1]))
        g.set_site(i, a / np.sqrt(4.0 * bonds[i]))
    g.move_center(0)
    g.set_site(0, g.site(0) / g.norm())
    for rep in range(2):
        c, t_copy = t(g.copy)
        _, t_l = t(lambda: c.move_center(n - 1))
        _, t_r = t(lambda: c.move_center(0))
        u = uniform_variates(5, 0, shots * n).reshape(shots, n)
        _, t_walk = t(lambda: c.sample_segment(0, n, u))
        _, t_all = t(lambda: P.sample(g, shots, 5))
        print(f"SAMPLE rep={rep} n={n} chi={chi} shots={shots}: copy {t_copy:.1f} ms, left sweep {t_l:.1f} ms, "
              f"right sweep {t_r:.1f} ms, walk {t_walk:.1f} ms, Sampler.sample {t_all:.1f} ms", flush=True)


if __name__ == "__main__":
    main()
