"""TEST INFRASTRUCTURE — NOT PRODUCT CODE.

ctypes wrapper around ``liboracle.so``, the Eigen-free C++ restatement of the
reference ``mpsim`` CPU path (see ``mps_oracle.hpp``). Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs import this
module, and only as the checker or the timed CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

# GateKind ordinals (circuit.hpp:26-31 / mps_oracle.hpp)
KINDS = ["h", "x", "y", "z", "s", "sdg", "t", "tdg", "rx", "ry", "rz", "u1", "u2", "u3",
         "cx", "cz", "swap", "u4"]
KIND = {k: i for i, k in enumerate(KINDS)}

I64 = C.c_int64
U64 = C.c_uint64
DP = C.POINTER(C.c_double)


def build(force: bool = False) -> str:
    srcs = ["mps_oracle.cpp", "oracle_capi.cpp", "mps_oracle.hpp"]
    newest = max(os.path.getmtime(os.path.join(_HERE, s)) for s in srcs)
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < newest:
        subprocess.run(["make", "-s", "-C", _HERE, "-B" if force else "all"], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        vp = C.c_void_p
        L.orc_last_error.restype = C.c_char_p
        for name in ["orc_state_new", "orc_state_random", "orc_state_copy", "orc_circuit_new",
                     "orc_circuit_brickwork", "orc_circuit_ghz", "orc_circuit_random", "orc_gates_new",
                     "orc_fuse", "orc_decompose", "orc_sampler_new"]:
            getattr(L, name).restype = vp
        L.orc_state_new.argtypes = [C.c_int]
        L.orc_state_random.argtypes = [C.c_int, I64, U64]
        L.orc_state_copy.argtypes = [vp]
        L.orc_state_free.argtypes = [vp]
        L.orc_state_n.argtypes = [vp]
        L.orc_state_bonds.argtypes = [vp, C.POINTER(I64)]
        L.orc_state_center.argtypes = [vp]
        L.orc_state_set_center.argtypes = [vp, C.c_int]
        L.orc_state_validate.argtypes = [vp]
        L.orc_get_site.argtypes = [vp, C.c_int, C.POINTER(I64), C.POINTER(I64), DP]
        L.orc_set_site.argtypes = [vp, C.c_int, I64, I64, DP]
        L.orc_apply_1q.argtypes = [vp, DP, C.c_int, DP, C.POINTER(I64), C.POINTER(C.c_int)]
        L.orc_apply_2q.argtypes = [vp, DP, C.c_int, C.c_int, C.c_int, I64, C.c_double, DP,
                                   C.POINTER(I64), C.POINTER(C.c_int)]
        L.orc_move_center.argtypes = [vp, C.c_int]
        L.orc_norm.argtypes = [vp, DP]
        L.orc_amplitude.argtypes = [vp, C.c_char_p, DP]
        L.orc_overlap.argtypes = [vp, vp, DP]
        L.orc_to_statevector.argtypes = [vp, C.c_int, DP]
        L.orc_svd.argtypes = [C.c_int, C.c_int, DP, I64, C.c_double, C.POINTER(I64), DP, DP, DP, DP]
        L.orc_truncation_rank.argtypes = [DP, I64, I64, C.c_double, DP]
        L.orc_truncation_rank.restype = I64
        L.orc_haar.argtypes = [C.c_int, U64, DP]
        L.orc_circuit_new.argtypes = [C.c_int]
        L.orc_circuit_free.argtypes = [vp]
        L.orc_circuit_add.argtypes = [vp, C.c_int, C.c_int, C.c_int, DP, C.c_int, DP]
        L.orc_circuit_brickwork.argtypes = [C.c_int, C.c_int, U64, C.c_int]
        L.orc_circuit_ghz.argtypes = [C.c_int]
        L.orc_circuit_random.argtypes = [C.c_int, C.c_int, U64, C.c_int]
        L.orc_circuit_size.argtypes = [vp]
        L.orc_circuit_n.argtypes = [vp]
        L.orc_circuit_get.argtypes = [vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                      C.POINTER(C.c_int), DP, C.POINTER(C.c_int)]
        L.orc_gate_matrix.argtypes = [C.c_int, C.c_int, C.c_int, DP, C.c_int, DP, DP]
        L.orc_gates_free.argtypes = [vp]
        L.orc_gates_size.argtypes = [vp]
        L.orc_gates_add.argtypes = [vp, C.c_int, C.c_int, DP]
        L.orc_gates_get.argtypes = [vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    C.POINTER(C.c_int), DP]
        L.orc_fuse.argtypes = [vp]
        L.orc_decompose.argtypes = [vp, C.c_int]
        L.orc_layerize.argtypes = [vp, C.POINTER(C.c_int)]
        L.orc_execute_serial.argtypes = [vp, vp, I64, C.c_double, C.c_int, DP, C.POINTER(I64), DP,
                                         C.POINTER(I64), C.POINTER(U64)]
        L.orc_execute_parallel.argtypes = [vp, vp, I64, C.c_double, C.c_int, DP, C.POINTER(I64), DP,
                                           C.POINTER(I64), C.POINTER(U64)]
        L.orc_sv_run.argtypes = [C.c_int, vp, DP]
        L.orc_sv_run_circuit.argtypes = [vp, DP]
        L.orc_sampler_new.argtypes = [vp, C.c_int, U64]
        L.orc_sampler_free.argtypes = [vp]
        L.orc_sample.argtypes = [vp, U64, U64, C.POINTER(C.c_int)]
        L.orc_sample_get.argtypes = [vp, C.c_int, C.c_char_p, C.POINTER(U64)]
        L.orc_sampler_hits.argtypes = [vp]
        L.orc_sampler_hits.restype = U64
        L.orc_sampler_cache_size.argtypes = [vp]
        L.orc_sampler_cache_size.restype = U64
        L.orc_sampler_clear.argtypes = [vp]
        L.orc_set_svd_backend.argtypes = [C.c_int]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class NumericError(OracleError):
    pass


def _check(rc):
    if rc != 0:
        msg = lib().orc_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        if rc == 3:
            raise NumericError(rc, msg)
        raise OracleError(rc, msg)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(DP)


def _cmat(u) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(u, dtype=np.complex128))


UNBOUNDED = (1 << 63) - 1


class Report:
    __slots__ = ("discarded_weight", "new_bond", "svd_count")

    def __init__(self, w, k, svd):
        self.discarded_weight, self.new_bond, self.svd_count = w, k, svd

    def __repr__(self):
        return f"Report(w={self.discarded_weight}, k={self.new_bond}, svd={self.svd_count})"


class MpsState:
    """Oracle MPS state (mps.hpp:33-75)."""

    def __init__(self, n: int | None = None, _handle=None):
        L = lib()
        if _handle is None:
            _handle = L.orc_state_new(int(n))
            if not _handle:
                raise ValueError(L.orc_last_error().decode())
        self._h = _handle

    @classmethod
    def random(cls, n, chi, seed):
        h = lib().orc_state_random(n, chi, seed)
        if not h:
            raise OracleError(4, lib().orc_last_error().decode())
        return cls(_handle=h)

    def copy(self):
        return MpsState(_handle=lib().orc_state_copy(self._h))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_state_free(self._h)
            self._h = None

    @property
    def n(self):
        return lib().orc_state_n(self._h)

    def bond_dims(self):
        out = np.zeros(self.n + 1, dtype=np.int64)
        lib().orc_state_bonds(self._h, out.ctypes.data_as(C.POINTER(I64)))
        return out

    def max_bond_dim(self):
        return int(self.bond_dims().max())

    @property
    def ortho_center(self):
        c = lib().orc_state_center(self._h)
        return None if c < 0 else c

    def set_ortho_center(self, c):
        lib().orc_state_set_center(self._h, -1 if c is None else int(c))

    def validate(self):
        _check(lib().orc_state_validate(self._h))

    def site(self, i) -> np.ndarray:
        dl, dr = I64(), I64()
        _check(lib().orc_get_site(self._h, i, C.byref(dl), C.byref(dr), None))
        out = np.zeros((dl.value, 2, dr.value), dtype=np.complex128)
        _check(lib().orc_get_site(self._h, i, C.byref(dl), C.byref(dr), _dp(out)))
        return out

    def set_site(self, i, t):
        t = _cmat(t)
        _check(lib().orc_set_site(self._h, i, t.shape[0], t.shape[2], _dp(t)))

    # gate application (gate_apply.hpp:48-78)
    def apply_1q(self, u, q):
        u = _cmat(u)
        w, k, s = C.c_double(), I64(), C.c_int()
        _check(lib().orc_apply_1q(self._h, _dp(u), q, C.byref(w), C.byref(k), C.byref(s)))
        return Report(w.value, k.value, s.value)

    def _apply_2q(self, u, q0, q1, method, max_bond, cutoff):
        u = _cmat(u)
        w, k, s = C.c_double(), I64(), C.c_int()
        mb = UNBOUNDED if max_bond in (None, 0) else int(max_bond)
        _check(lib().orc_apply_2q(self._h, _dp(u), q0, q1, method, mb, float(cutoff), C.byref(w),
                                  C.byref(k), C.byref(s)))
        return Report(w.value, k.value, s.value)

    def apply_2q_local(self, u, q, max_bond=None, cutoff=0.0):
        return self._apply_2q(u, q, q + 1, 0, max_bond, cutoff)

    def apply_2q_swap(self, u, q0, q1, max_bond=None, cutoff=0.0):
        return self._apply_2q(u, q0, q1, 1, max_bond, cutoff)

    def apply_2q_bondprop(self, u, q0, q1, max_bond=None, cutoff=0.0):
        return self._apply_2q(u, q0, q1, 2, max_bond, cutoff)

    # queries (mps.hpp:79-100)
    def move_center(self, c):
        _check(lib().orc_move_center(self._h, c))

    def norm(self):
        v = C.c_double()
        _check(lib().orc_norm(self._h, C.byref(v)))
        return v.value

    def amplitude(self, bits: str):
        out = np.zeros(2)
        _check(lib().orc_amplitude(self._h, bits.encode(), _dp(out)))
        return complex(out[0], out[1])

    def overlap(self, other: "MpsState"):
        out = np.zeros(2)
        _check(lib().orc_overlap(self._h, other._h, _dp(out)))
        return complex(out[0], out[1])

    def to_statevector(self, max_qubits=20):
        n = self.n
        if n > max_qubits:
            raise ValueError("statevector export capped")
        out = np.zeros(1 << n, dtype=np.complex128)
        _check(lib().orc_to_statevector(self._h, max_qubits, _dp(out)))
        return out


def svd(m, max_rank=None, cutoff=0.0):
    m = _cmat(m)
    r, c = m.shape
    mn = min(r, c)
    s = np.zeros(mn)
    u = np.zeros((r, mn), dtype=np.complex128)
    v = np.zeros((mn, c), dtype=np.complex128)
    k, w = I64(), C.c_double()
    mr = UNBOUNDED if max_rank is None else int(max_rank)
    _check(lib().orc_svd(r, c, _dp(m), mr, float(cutoff), C.byref(k), _dp(s), _dp(u), _dp(v), C.byref(w)))
    kk = k.value
    return u.reshape(-1)[: r * kk].reshape(r, kk), s[:kk], v.reshape(-1)[: kk * c].reshape(kk, c), w.value


def set_svd_backend(name: str):
    """'zgesdd' (default; divide and conquer, Eigen BDCSVD's family), 'zgesvj'
    (one-sided Jacobi: an independent check of the first) or 'zgesvd'
    (bidiagonal QR iteration)."""
    lib().orc_set_svd_backend({"zgesdd": 0, "zgesvj": 1, "zgesvd": 2}[name])


def truncation_rank(s, max_rank=None, cutoff=0.0):
    s = np.ascontiguousarray(s, dtype=np.float64)
    w = C.c_double()
    mr = UNBOUNDED if max_rank is None else int(max_rank)
    k = lib().orc_truncation_rank(_dp(s), len(s), mr, float(cutoff), C.byref(w))
    return k, w.value


def haar_unitary(dim, seed):
    out = np.zeros((dim, dim), dtype=np.complex128)
    lib().orc_haar(dim, seed, _dp(out))
    return out


class Circuit:
    """Primitive op list (circuit.hpp:61-66)."""

    def __init__(self, n=None, _handle=None):
        self._h = _handle if _handle is not None else lib().orc_circuit_new(n)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_circuit_free(self._h)
            self._h = None

    @classmethod
    def brickwork(cls, n, depth, seed, haar=False):
        h = lib().orc_circuit_brickwork(n, depth, seed, 1 if haar else 0)
        if not h:
            raise ValueError(lib().orc_last_error().decode())
        return cls(_handle=h)

    @classmethod
    def ghz(cls, n):
        return cls(_handle=lib().orc_circuit_ghz(n))

    @classmethod
    def random(cls, n, gates, seed, nonlocal_=True):
        return cls(_handle=lib().orc_circuit_random(n, gates, seed, 1 if nonlocal_ else 0))

    def add(self, kind, q0, q1=-1, params=(), matrix=None):
        p = np.ascontiguousarray(params, dtype=np.float64)
        m = _cmat(matrix) if matrix is not None else np.zeros((4, 4), dtype=np.complex128)
        _check(lib().orc_circuit_add(self._h, KIND[kind], q0, q1, _dp(p), len(p), _dp(m)))
        return self

    @property
    def n(self):
        return lib().orc_circuit_n(self._h)

    def __len__(self):
        return lib().orc_circuit_size(self._h)

    def ops(self):
        out = []
        kind, q0, q1, np_ = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        params = np.zeros(3)
        for i in range(len(self)):
            _check(lib().orc_circuit_get(self._h, i, C.byref(kind), C.byref(q0), C.byref(q1), _dp(params),
                                         C.byref(np_)))
            out.append((KINDS[kind.value], q0.value, q1.value, tuple(params[: np_.value])))
        return out

    def fuse(self) -> "GateList":
        return GateList(_handle=lib().orc_fuse(self._h))

    def statevector(self):
        out = np.zeros(1 << self.n, dtype=np.complex128)
        _check(lib().orc_sv_run_circuit(self._h, _dp(out)))
        return out


def gate_matrix(kind, q0=0, q1=-1, params=(), u4=None):
    p = np.ascontiguousarray(params, dtype=np.float64)
    m = _cmat(u4) if u4 is not None else np.zeros((4, 4), dtype=np.complex128)
    dim = 4 if q1 >= 0 else 2
    out = np.zeros((dim, dim), dtype=np.complex128)
    _check(lib().orc_gate_matrix(KIND[kind], q0, q1, _dp(p), len(p), _dp(m), _dp(out)))
    return out


class GateList:
    """Fused-gate list (circuit.hpp:71-81)."""

    def __init__(self, gates=None, _handle=None):
        self._h = _handle if _handle is not None else lib().orc_gates_new()
        for g in gates or []:
            self.add(*g)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_gates_free(self._h)
            self._h = None

    def add(self, q0, q1, m):
        m = _cmat(m)
        _check(lib().orc_gates_add(self._h, q0, q1, _dp(m)))

    def __len__(self):
        return lib().orc_gates_size(self._h)

    def gates(self):
        """[(q0, q1, flipped, matrix)]"""
        out = []
        q0, q1, fl = C.c_int(), C.c_int(), C.c_int()
        for i in range(len(self)):
            m = np.zeros(16, dtype=np.complex128)
            _check(lib().orc_gates_get(self._h, i, C.byref(q0), C.byref(q1), C.byref(fl), _dp(m)))
            dim = 4 if q1.value >= 0 else 2
            out.append((q0.value, q1.value, bool(fl.value), m[: dim * dim].reshape(dim, dim).copy()))
        return out

    def decompose_nonlocal(self, n) -> "GateList":
        h = lib().orc_decompose(self._h, n)
        if not h:
            raise ValueError(lib().orc_last_error().decode())
        return GateList(_handle=h)

    def layer_of(self):
        out = np.zeros(max(1, len(self)), dtype=np.int32)
        nl = lib().orc_layerize(self._h, out.ctypes.data_as(C.POINTER(C.c_int)))
        if nl < 0:
            raise ValueError(lib().orc_last_error().decode())
        return out[: len(self)], nl

    def statevector(self, n):
        out = np.zeros(1 << n, dtype=np.complex128)
        _check(lib().orc_sv_run(n, self._h, _dp(out)))
        return out


def _exec(fn, state, gates, max_bond, cutoff, extra):
    ng = len(gates)
    tw, pk, wall = C.c_double(), I64(), U64()
    gw = np.zeros(max(ng, 1))
    gk = np.zeros(max(ng, 1), dtype=np.int64)
    mb = UNBOUNDED if max_bond in (None, 0) else int(max_bond)
    _check(fn(state._h, gates._h, mb, float(cutoff), extra, C.byref(tw), C.byref(pk), _dp(gw),
              gk.ctypes.data_as(C.POINTER(I64)), C.byref(wall)))
    return dict(total_discarded_weight=tw.value, peak_bond=pk.value, gate_w=gw[:ng], gate_k=gk[:ng],
                wall_ns=wall.value)


def execute_serial(state, gates, max_bond=None, cutoff=0.0, bondprop=False):
    return _exec(lib().orc_execute_serial, state, gates, max_bond, cutoff, 1 if bondprop else 0)


def execute_parallel(state, gates, max_bond=None, cutoff=0.0, workers=1):
    """Layerizes ``gates`` (must be local) and runs them; reports in layer-plan order."""
    return _exec(lib().orc_execute_parallel, state, gates, max_bond, cutoff, int(workers))


class Sampler:
    def __init__(self, state, memoize=True, cache_cap=0):
        self._h = lib().orc_sampler_new(state._h, 1 if memoize else 0, cache_cap)
        if not self._h:
            raise NumericError(3, lib().orc_last_error().decode())
        self._n = state.n

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_sampler_free(self._h)
            self._h = None

    def sample(self, shots, seed):
        u = C.c_int()
        _check(lib().orc_sample(self._h, shots, seed, C.byref(u)))
        out = {}
        buf = C.create_string_buffer(self._n + 1)
        cnt = U64()
        for i in range(u.value):
            lib().orc_sample_get(self._h, i, buf, C.byref(cnt))
            out[buf.raw[: self._n].decode()] = cnt.value
        return out

    @property
    def cache_hits(self):
        return lib().orc_sampler_hits(self._h)

    @property
    def cache_size(self):
        return lib().orc_sampler_cache_size(self._h)

    def clear_cache(self):
        lib().orc_sampler_clear(self._h)
