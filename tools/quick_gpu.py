"""Quick GPU parity probe (dev tool): GPU engine vs CPU oracle."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
import paper_2601_04422_b200 as P

def dense2(pre, u, q0, q1, n):
    psi = pre.reshape([2]*n)
    psi = np.moveaxis(psi, [q0, q1], [0, 1]).reshape(4, -1)
    psi = (u @ psi).reshape([2, 2] + [2]*(n-2))
    return np.moveaxis(psi, [0, 1], [q0, q1]).reshape(-1)

cx = np.array([[1,0,0,0],[0,1,0,0],[0,0,0,1],[0,0,1,0]], dtype=complex)
s = P.MpsState(2); r = s.apply_2q_local(cx, 0); print("cx|00>", r, s.amplitude("00"))
h = np.array([[1,1],[1,-1]])/np.sqrt(2)
s = P.MpsState(2); s.apply_1q(h, 0); r = s.apply_2q_local(cx, 0); print("bell", r, s.to_statevector())
for seed in range(1, 7):
    o = O.MpsState.random(6, 6, 100 + seed)
    g = P.MpsState(6)
    for i in range(6): g.set_site(i, o.site(i))
    pre = o.to_statevector()
    u = O.haar_unitary(4, 17*seed); q = seed % 5
    r = g.apply_2q_local(u, q); ro = o.apply_2q_local(u, q)
    print(seed, r, ro, np.abs(g.to_statevector() - dense2(pre, u, q, q+1, 6)).max(), g.norm(), g.bond_dims(), o.bond_dims())
# truncation
for seed in range(1, 4):
    o = O.MpsState.random(8, 16, 300 + seed)
    g = P.MpsState(8)
    for i in range(8): g.set_site(i, o.site(i))
    u = O.haar_unitary(4, 5*seed)
    r = g.apply_2q_local(u, 3, max_bond=5, cutoff=1e-3); ro = o.apply_2q_local(u, 3, max_bond=5, cutoff=1e-3)
    print("trunc", r, ro, abs(g.overlap(g) - 1), abs(abs(g.to_statevector().conj() @ o.to_statevector()) - 1))
# brickwork C2 small
c = O.Circuit.brickwork(16, 8, 4242, haar=True); gl = c.fuse()
gates = [(q0, q1, m) for (q0, q1, f, m) in gl.gates()]
o = O.MpsState(16); t0 = time.time(); ro = O.execute_serial(o, gl, 16, 1e-12); t1 = time.time()
g = P.MpsState(16); rg = P.execute(g, gates, 16, 1e-12); t2 = time.time()
print("brick", ro['peak_bond'], rg['peak_bond'], (ro['gate_k'] == rg['gate_k']).all(), ro['total_discarded_weight'], rg['total_discarded_weight'], t1-t0, t2-t1, rg['layers'], rg['kernel_launches'])
print("fid", abs(np.vdot(o.to_statevector(), g.to_statevector())))
