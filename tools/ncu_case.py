"""Small fixed case for ncu: one brick layer of 8 Haar gates at chi=512."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2601_04422_b200 as P
exec(open('tools/perf_probe.py').read().split("chi = int")[0])
import os
chi, ngates = int(os.environ.get('CHI', '512')), int(os.environ.get('NGATES', '8'))
rng = np.random.default_rng(1)
lg = int(np.log2(chi)); n = 2 * (lg + 1) + 2 * ngates
s, bonds = saturated_state(n, chi, rng)
start = lg + 1 + ((lg + 1) % 2)
gates = [(q, q + 1, haar4(rng)) for q in range(start, start + 2 * ngates, 2)]
r = s.apply_layer(gates, max_bond=chi, cutoff=1e-12)
print("ok", s.counters())
