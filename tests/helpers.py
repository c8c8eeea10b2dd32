"""Shared test helpers: independent numpy restatements used as a second oracle."""
import numpy as np

HAD = np.array([[1, 1], [1, -1]], dtype=complex) / np.sqrt(2)
PX = np.array([[0, 1], [1, 0]], dtype=complex)
PZ = np.array([[1, 0], [0, -1]], dtype=complex)
CX = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=complex)
SWAP = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=complex)


def dense_apply_1q(psi, u, q, n):
    t = np.moveaxis(psi.reshape([2] * n), q, 0).reshape(2, -1)
    t = (u @ t).reshape([2] * n)
    return np.moveaxis(t, 0, q).reshape(-1)


def dense_apply_2q(psi, u, q0, q1, n):
    """u in the (q0, q1) basis: row = 2*bit(q0) + bit(q1) (circuit.hpp:20-22)."""
    t = np.moveaxis(psi.reshape([2] * n), [q0, q1], [0, 1]).reshape(4, -1)
    t = (u @ t).reshape([2, 2] + [2] * (n - 2))
    return np.moveaxis(t, [0, 1], [q0, q1]).reshape(-1)


def max_dev(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max())


def phase_aligned_max_deviation(a, b):
    """tests/support/test_util.cpp:135-156."""
    a, b = np.asarray(a), np.asarray(b)
    p = int(np.argmax(np.abs(a)))
    phase = 1.0
    if abs(a[p]) > 0 and abs(b[p]) > 0:
        phase = a[p] / b[p]
        phase /= abs(phase)
    return float(np.abs(a - phase * b).max())


def bits_of(index, n):
    return format(index, f"0{n}b")


def copy_state_to_gpu(P, ostate, chi_hint=16):
    """Import an oracle state site by site (MpsState::site(i) writes, test_util.cpp:104-106)."""
    n = ostate.n
    g = P.MpsState(n, chi_hint=chi_hint)
    for i in range(n):
        g.set_site(i, ostate.site(i))
    c = ostate.ortho_center
    g.set_ortho_center(c)
    return g


def gate_tuples(gl):
    return [(q0, q1, m) for (q0, q1, _f, m) in gl.gates()]


def rel(a, b):
    a, b = complex(a), complex(b)
    d = max(abs(a), abs(b))
    return 0.0 if d == 0 else abs(a - b) / d


class MT19937_64:
    """std::mt19937_64 (the reference's generator engine, generators.cpp:31-33)."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.i = 312

    def __call__(self):
        if self.i >= 312:
            mt = self.mt
            for k in range(312):
                y = (mt[k] & 0xFFFFFFFF80000000) | (mt[(k + 1) % 312] & 0x7FFFFFFF)
                v = mt[(k + 156) % 312] ^ (y >> 1)
                if y & 1:
                    v ^= 0xB5026F5AA96619E9
                mt[k] = v
            self.i = 0
        x = self.mt[self.i]
        self.i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & 0xFFFFFFFFFFFFFFFF

    def unit(self):
        return (self() >> 11) * 2.0 ** -53
