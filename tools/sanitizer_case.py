"""Small case for compute-sanitizer (racecheck / memcheck / synccheck): one
brick layer of 4 Haar gates at chi = 64 through the persistent Jacobi sweep
kernel, the TMA theta kernel, QR preconditioning, the split epilogue, then a
centre move and a short sample. Prints 'ok' with the counters."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_04422_b200 as P  # noqa: E402


def haar4(rng):
    z = (rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))) / np.sqrt(2)
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


chi = int(os.environ.get("CHI", "64"))
n = 16
rng = np.random.default_rng(5)
bonds = [min(chi, 2 ** min(i, n - i)) for i in range(n + 1)]
s = P.MpsState(n, chi_hint=chi)
for i in range(n):
    t = rng.standard_normal((bonds[i], 2, bonds[i + 1])) + 1j * rng.standard_normal((bonds[i], 2, bonds[i + 1]))
    s.set_site(i, t / np.sqrt(4.0 * bonds[i]))
gates = [(q, q + 1, haar4(rng)) for q in range(5, 13, 2)]
r = s.apply_layer(gates, max_bond=chi, cutoff=1e-12)
s.move_center(8)
s.set_site(8, s.site(8) / s.norm())
counts = P.sample(s, 200, 3)
print("ok", [x.new_bond for x in r], len(counts), s.counters())
