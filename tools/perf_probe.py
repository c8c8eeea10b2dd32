"""Dev perf probe: one brick layer of Haar gates on a chi-saturated random MPS."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_2601_04422_b200 as P

def haar4(rng):
    z = (rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))) / np.sqrt(2)
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))

def saturated_state(n, chi, rng):
    s = P.MpsState(n, chi_hint=chi)
    bonds = [min(chi, 2 ** min(i, n - i)) for i in range(n + 1)]
    for i in range(n):
        dl, dr = bonds[i], bonds[i + 1]
        t = (rng.standard_normal((dl, 2, dr)) + 1j * rng.standard_normal((dl, 2, dr))) / np.sqrt(4.0 * dl)
        s.set_site(i, t)
    return s, bonds

chi = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ngates = int(sys.argv[2]) if len(sys.argv) > 2 else 8
rng = np.random.default_rng(1)
lg = int(np.log2(chi))
n = 2 * (lg + 1) + 2 * ngates
s, bonds = saturated_state(n, chi, rng)
start = lg + 1 + ((lg + 1) % 2)
gates = [(q, q + 1, haar4(rng)) for q in range(start, start + 2 * ngates, 2)]
print("n", n, "gates", len(gates), "dims", [(bonds[q], bonds[q+1], bonds[q+2]) for q, _, _ in gates[:2]])
for rep in range(3):
    s.reset_counters()
    t0 = time.time()
    r = s.apply_layer(gates, max_bond=chi, cutoff=1e-12)
    t1 = time.time()
    c = s.counters()
    print(f"rep {rep}: {t1-t0:.3f}s  {len(gates)/(t1-t0):.1f} gates/s  sweeps {c['sweeps']} launches {c['launches']} k={[x.new_bond for x in r[:4]]} w={r[0].discarded_weight:.3e}")
