"""Numpy emulation of the GPU block one-sided Jacobi (W = 16, round-robin
tournament over block pairs, de Rijk ordering per sweep, ONE cyclic inner
sweep of 2x2 complex rotations per pair visit, eigenvectors unsorted), used to
decide algorithmic variants before writing kernels. Counts outer sweeps to the
GPU's convergence test (all relative off-diagonals <= 4 eps * 32).

  python tools/emu_jacobi.py CHI VARIANT
    VARIANT: plain   Jacobi on theta's columns
             qr      Jacobi on R^H, theta = Q R (what qr_pre.cu does)
             qrcp    Jacobi on R^H of a column-pivoted QR
             qr2     Jacobi on R2^H, R^H = Q2 R2 (two QR steps); qr3, qr4 likewise
             cross   plain, cross-block-only inner sweeps while the measured
                     rms relative off-norm of the previous sweep > 0.35
Measured (chi = 512, theta 1024 x 1024 from a saturated random MPS):
plain 14 rotating sweeps, qr 11, qrcp 10, qr2 9; cross: no extra sweep.
"""
import sys

import numpy as np
import scipy.linalg as sl

W = int(__import__("os").environ.get("EMU_W", "16"))
EPS = 2.220446049250313e-16


def theta(chi, rng):
    def haar(n):
        z = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2)
        q, r = np.linalg.qr(z)
        return q * (np.diag(r) / np.abs(np.diag(r)))
    a = (rng.standard_normal((chi, 2, chi)) + 1j * rng.standard_normal((chi, 2, chi))) / np.sqrt(4 * chi)
    b = (rng.standard_normal((chi, 2, chi)) + 1j * rng.standard_normal((chi, 2, chi))) / np.sqrt(4 * chi)
    u = haar(4).reshape(2, 2, 2, 2)
    t = np.einsum('asb,btc->astc', a, b)
    return np.einsum('stuv,auvc->astc', u, t).reshape(2 * chi, 2 * chi)


def rr(nb):
    pl, rounds = list(range(nb)), []
    for _ in range(nb - 1):
        rounds.append([(pl[k], pl[nb - 1 - k]) for k in range(nb // 2)])
        pl = [pl[0]] + [pl[-1]] + pl[1:-1]
    return rounds


def inner_sweep(G, cross):
    """One cyclic sweep of 2x2 rotations (all pairs, or cross-block pairs
    only) on a batch of Hermitian 2W x 2W Grams; returns the accumulated R."""
    G = G.copy()
    nbat, k, _ = G.shape
    h = k // 2
    V = np.broadcast_to(np.eye(k, dtype=complex), G.shape).copy()
    steps = [[(p, h + (p + s) % h) for p in range(h)] for s in range(h)] if cross else rr(k)
    for stp in steps:
        p = np.array([x for x, _ in stp])
        q = np.array([y for _, y in stp])
        M = np.empty((nbat, len(p), 2, 2), complex)
        M[:, :, 0, 0], M[:, :, 1, 1] = G[:, p, p], G[:, q, q]
        M[:, :, 0, 1], M[:, :, 1, 0] = G[:, p, q], G[:, q, p]
        _, J = np.linalg.eigh(M)
        swap = np.abs(J[..., 0, 0]) < np.abs(J[..., 0, 1])  # |cos| >= |sin| (UBC)
        J[swap] = J[swap][..., ::-1]
        for arr, both in ((G, True), (V, False)):
            cp, cq = arr[:, :, p].copy(), arr[:, :, q].copy()
            arr[:, :, p] = cp * J[:, None, :, 0, 0] + cq * J[:, None, :, 1, 0]
            arr[:, :, q] = cp * J[:, None, :, 0, 1] + cq * J[:, None, :, 1, 1]
            if both:
                rp, rq = arr[:, p, :].copy(), arr[:, q, :].copy()
                arr[:, p, :] = J[:, :, 0, 0, None].conj() * rp + J[:, :, 1, 0, None].conj() * rq
                arr[:, q, :] = J[:, :, 0, 1, None].conj() * rp + J[:, :, 1, 1, None].conj() * rq
    return V


def run(X, fro2, cross_policy=False, max_sweeps=40):
    n = X.shape[1]
    nb = n // W
    tol = 4 * EPS * 32
    floor = (64 * EPS) ** 2 * fro2
    rms_prev = None
    for sweep in range(max_sweeps):
        G = X.conj().T @ X
        d2 = np.real(np.diag(G))
        R = np.abs(G) / np.sqrt(np.outer(d2, d2))
        noise = d2 <= floor
        R[noise, :] = 0
        R[:, noise] = 0
        np.fill_diagonal(R, 0)
        print(f"sweep {sweep}: max rel off {R.max():.3e}", flush=True)
        if R.max() <= tol:
            return sweep
        X = X[:, np.argsort(-np.linalg.norm(X, axis=0))]
        cross = cross_policy and rms_prev is not None and rms_prev > 0.35
        acc = 0.0
        for pairs in rr(nb):
            idx = np.array([np.r_[i * W:(i + 1) * W, j * W:(j + 1) * W] for i, j in pairs])
            P = X[:, idx].transpose(1, 0, 2)
            Gp = P.conj().transpose(0, 2, 1) @ P
            d = np.real(np.einsum('pii->pi', Gp))
            ok = (d[:, :W, None] > floor) & (d[:, None, W:] > floor)
            acc += (np.abs(Gp[:, :W, W:]) ** 2 / (d[:, :W, None] * d[:, None, W:]) * ok).sum()
            X[:, idx] = (P @ inner_sweep(Gp, cross)).transpose(1, 0, 2)
        rms_prev = np.sqrt(2 * acc / n)
    return max_sweeps


def main():
    chi = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    variant = sys.argv[2] if len(sys.argv) > 2 else "plain"
    th = theta(chi, np.random.default_rng(1))
    fro2 = np.linalg.norm(th) ** 2
    if variant in ("plain", "cross"):
        X = th.copy()
    elif variant in ("mp32", "mpgram", "mpgram32", "mp16"):
        # mixed-precision preconditioner: an approximate right singular basis V0,
        # made exactly unitary by an FP64 QR, then Jacobi on theta Q
        if variant == "mp32":
            V0 = np.linalg.svd(th.astype(np.complex64))[2].conj().T
        elif variant == "mp16":
            t16 = th + 1e-4 * np.linalg.norm(th, 2) * (np.random.default_rng(5).standard_normal(th.shape)) / np.sqrt(th.shape[0])
            V0 = np.linalg.svd(t16)[2].conj().T
        elif variant == "mpgram":
            V0 = np.linalg.eigh(th.conj().T @ th)[1][:, ::-1]
        else:
            g = (th.conj().T @ th).astype(np.complex64)
            V0 = np.linalg.eigh(g)[1][:, ::-1]
        Q = np.linalg.qr(V0.astype(np.complex128))[0]
        X = th @ Q
    elif variant == "qrcp":
        X = sl.qr(th, pivoting=True, mode='economic')[1].conj().T.copy()
    elif variant == "qrcp2":  # Drmac-Veselic: QRCP, then an (unpivoted) QR of R^H
        X = sl.qr(th, pivoting=True, mode='economic')[1].conj().T.copy()
        X = np.linalg.qr(X)[1].conj().T.copy()
    else:
        X = np.linalg.qr(th)[1].conj().T.copy()
        for _ in range({"qr2": 1, "qr3": 2, "qr4": 3}.get(variant, 0)):
            X = np.linalg.qr(X)[1].conj().T.copy()
    sweeps = run(X, fro2, cross_policy=variant == "cross")
    print(f"{variant}: converged after {sweeps} rotating sweeps")


if __name__ == "__main__":
    main()
