"""Host-side mirror of the reference simulator API over the C ABI.

Names, argument meaning and error behaviour follow the reference ``mpsim``
C++ API (``include/mpsim/mps.hpp``, ``gate_apply.hpp``, ``executor.hpp``,
``sampler.hpp``): ``std::invalid_argument`` -> ``ValueError``,
``NumericError`` -> ``native.NumericError``, ``std::logic_error`` ->
``native.LogicError``. All state lives in HBM; every operation runs on the GPU.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import native as N
from .native import check

_DP = N.DP


def _cm(u, dim) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(u, dtype=np.complex128))
    if a.shape != (dim, dim):
        raise ValueError(f"gate matrix must be {dim}x{dim}")
    return a


def _policy(max_bond=None, cutoff=0.0) -> N.Policy:
    mb = N.UNBOUNDED if max_bond is None else int(max_bond)
    return N.Policy(mb, float(cutoff))


def make_gates(gates) -> "C.Array":
    """[(q0, q1, matrix)] -> Gate array (q1 = -1 for one-qubit gates)."""
    arr = (N.Gate * max(1, len(gates)))()
    for i, (q0, q1, m) in enumerate(gates):
        dim = 2 if q1 is None or q1 < 0 else 4
        a = _cm(m, dim).reshape(-1)
        arr[i].q0 = int(q0)
        arr[i].q1 = -1 if dim == 2 else int(q1)
        flat = np.zeros(32)
        flat[: 2 * dim * dim] = a.view(np.float64)
        C.memmove(arr[i].u, flat.ctypes.data, 32 * 8)
    return arr


def svd(m, max_rank=None, cutoff=0.0, device=0):
    """Truncated SVD (svd.hpp:79-110) on the GPU: returns (u, s, vdag, w)."""
    a = np.ascontiguousarray(np.asarray(m, dtype=np.complex128))
    if a.ndim != 2:
        raise ValueError("svd requires a rank-2 tensor")
    r, c = a.shape
    mn = min(r, c)
    s = np.zeros(mn)
    u = np.zeros(r * mn, dtype=np.complex128)
    v = np.zeros(mn * c, dtype=np.complex128)
    k, w = N.I64(), C.c_double()
    mr = N.UNBOUNDED if max_rank is None else int(max_rank)
    check(N.lib().mpsim_gpu_svd(r, c, a.ctypes.data_as(_DP), mr, float(cutoff), int(device), C.byref(k),
                                s.ctypes.data_as(_DP), u.ctypes.data_as(_DP), v.ctypes.data_as(_DP), C.byref(w)))
    kk = k.value
    return u[: r * kk].reshape(r, kk), s[:kk], v[: kk * c].reshape(kk, c), w.value


class MpsState:
    """MpsState (mps.hpp:33-75), resident on one GPU."""

    def __init__(self, n: int | None = None, chi_hint: int = 16, device: int = 0, _handle=None):
        L = N.lib()
        if _handle is None:
            h = C.c_void_p()
            check(L.mpsim_gpu_state_create(int(n), int(chi_hint), int(device), C.byref(h)))
            _handle = h
        self._h = _handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and N._lib is not None and not getattr(self, "_borrowed", False):
            N._lib.mpsim_gpu_state_destroy(h)
            self._h = None

    def copy(self) -> "MpsState":
        h = C.c_void_p()
        check(N.lib().mpsim_gpu_state_copy(self._h, C.byref(h)))
        return MpsState(_handle=h)

    # ---- bookkeeping
    @property
    def n(self) -> int:
        v = N.I32()
        check(N.lib().mpsim_gpu_num_qubits(self._h, C.byref(v)))
        return v.value

    num_qubits = n

    def bond_dims(self) -> np.ndarray:
        out = np.zeros(self.n + 1, dtype=np.int64)
        check(N.lib().mpsim_gpu_bond_dims(self._h, out.ctypes.data_as(C.POINTER(N.I64))))
        return out

    def bond_dim(self, i):
        return int(self.bond_dims()[i])

    def max_bond_dim(self) -> int:
        return int(self.bond_dims().max())

    def set_bond_dim(self, i, d):
        check(N.lib().mpsim_gpu_set_bond_dim(self._h, int(i), int(d)))

    @property
    def chi_capacity(self) -> int:
        v = N.I64()
        check(N.lib().mpsim_gpu_chi_capacity(self._h, C.byref(v)))
        return v.value

    @property
    def ortho_center(self):
        v = N.I32()
        check(N.lib().mpsim_gpu_ortho_center(self._h, C.byref(v)))
        return None if v.value < 0 else v.value

    def set_ortho_center(self, c):
        check(N.lib().mpsim_gpu_set_ortho_center(self._h, -1 if c is None else int(c)))

    def validate(self):
        check(N.lib().mpsim_gpu_validate(self._h))

    def site(self, i) -> np.ndarray:
        dl, dr = N.I64(), N.I64()
        check(N.lib().mpsim_gpu_get_site(self._h, int(i), C.byref(dl), C.byref(dr), None))
        out = np.zeros((dl.value, 2, dr.value), dtype=np.complex128)
        check(N.lib().mpsim_gpu_get_site(self._h, int(i), C.byref(dl), C.byref(dr), out.ctypes.data_as(_DP)))
        return out

    def set_site(self, i, t):
        t = np.ascontiguousarray(np.asarray(t, dtype=np.complex128))
        if t.ndim != 3 or t.shape[1] != 2:
            raise ValueError("site must be a (left, 2, right) tensor")
        check(N.lib().mpsim_gpu_set_site(self._h, int(i), t.shape[0], t.shape[2], t.ctypes.data_as(_DP)))

    # ---- shard plumbing (multi-GPU chains)
    def set_open_boundaries(self, open_=True):
        check(N.lib().mpsim_gpu_set_open_boundaries(self._h, 1 if open_ else 0))

    def site_slot(self, i):
        """(device pointer, chi) of site i's padded (chi, 2, chi) slot."""
        p, chi = C.c_void_p(), N.I64()
        check(N.lib().mpsim_gpu_site_slot(self._h, int(i), C.byref(p), C.byref(chi)))
        return p.value, chi.value

    def set_site_dims(self, i, dl, dr):
        check(N.lib().mpsim_gpu_set_site_dims(self._h, int(i), int(dl), int(dr)))

    def total_elements(self) -> int:
        b = self.bond_dims()
        return int(sum(b[i] * 2 * b[i + 1] for i in range(self.n)))

    # ---- gate application (gate_apply.hpp:48-78)
    def apply_1q(self, u, q):
        u = _cm(u, 2)
        r = N.Report()
        check(N.lib().mpsim_gpu_apply_1q(self._h, u.ctypes.data_as(_DP), int(q), C.byref(r)))
        return r

    def _apply_2q(self, u, q0, q1, method, max_bond, cutoff):
        u = _cm(u, 4)
        r = N.Report()
        p = _policy(max_bond, cutoff)
        check(N.lib().mpsim_gpu_apply_2q(self._h, u.ctypes.data_as(_DP), int(q0), int(q1), method, C.byref(p),
                                         C.byref(r)))
        return r

    def apply_2q_local(self, u, q, max_bond=None, cutoff=0.0):
        if q < 0 or q + 1 >= self.n:
            raise ValueError(f"adjacent pair ({q},{q + 1}) out of range")
        return self._apply_2q(u, q, q + 1, N.NONLOCAL_SWAP, max_bond, cutoff)

    def apply_2q_swap(self, u, q0, q1, max_bond=None, cutoff=0.0):
        return self._apply_2q(u, q0, q1, N.NONLOCAL_SWAP, max_bond, cutoff)

    def apply_2q_bondprop(self, u, q0, q1, max_bond=None, cutoff=0.0):
        return self._apply_2q(u, q0, q1, N.NONLOCAL_BONDPROP, max_bond, cutoff)

    def apply_layer(self, gates, max_bond=None, cutoff=0.0):
        """One batched launch for disjoint local gates [(q0, q1, matrix)]."""
        arr = make_gates(gates)
        reps = (N.Report * max(1, len(gates)))()
        p = _policy(max_bond, cutoff)
        check(N.lib().mpsim_gpu_apply_layer(self._h, arr, len(gates), C.byref(p), reps))
        return list(reps)[: len(gates)]

    # ---- queries (mps.hpp:79-100)
    def norm(self) -> float:
        v = C.c_double()
        check(N.lib().mpsim_gpu_norm(self._h, C.byref(v)))
        return v.value

    def amplitudes(self, bitstrings) -> np.ndarray:
        n = self.n
        for b in bitstrings:
            if len(b) != n:
                raise ValueError(f"bit string length {len(b)} does not match qubit count {n}")
        buf = "".join(bitstrings).encode()
        out = np.zeros(2 * len(bitstrings))
        check(N.lib().mpsim_gpu_amplitudes(self._h, buf, len(bitstrings), out.ctypes.data_as(_DP)))
        return out.view(np.complex128)

    def amplitude(self, bits: str) -> complex:
        return complex(self.amplitudes([bits])[0])

    def overlap(self, other: "MpsState") -> complex:
        out = np.zeros(2)
        check(N.lib().mpsim_gpu_overlap(self._h, other._h, out.ctypes.data_as(_DP)))
        return complex(out[0], out[1])

    # ---- move_center pieces (site-sharded chains)
    def sweep_left(self, i0, i1):
        """Left steps on sites [i0, i1) (mps.cpp:69-80)."""
        check(N.lib().mpsim_gpu_sweep_left(self._h, int(i0), int(i1)))

    def sweep_right(self, i0, i1):
        """Right steps on sites i1 down to i0 >= 1 (mps.cpp:84-95)."""
        check(N.lib().mpsim_gpu_sweep_right(self._h, int(i0), int(i1)))

    def site_norm2(self, i) -> float:
        v = C.c_double()
        check(N.lib().mpsim_gpu_site_norm2(self._h, int(i), C.byref(v)))
        return v.value

    def sample_segment(self, i0, i1, u, env_in=None, node_in=None):
        """The sampler's site walk over sites [i0, i1) of a canonicalised
        state: u (shots x (i1 - i0)) variates; env_in (U x D_left) / node_in
        (shots) the prefixes from the left. Returns (env_out U' x D_right,
        node_out, bits) with bits a list of per-shot strings."""
        u = np.ascontiguousarray(u, dtype=np.float64)
        shots, w = u.shape
        dims = self.bond_dims()
        ein = nin = None
        uin = 1
        if env_in is not None:
            ein = np.ascontiguousarray(env_in, dtype=np.complex128)
            uin = ein.shape[0]
            nin = np.ascontiguousarray(node_in, dtype=np.int32)
        dr = int(dims[i1])
        eout = np.zeros((shots, dr), dtype=np.complex128)
        nout = np.zeros(shots, dtype=np.int32)
        bits = C.create_string_buffer(shots * w)
        uo = N.I32()
        check(N.lib().mpsim_gpu_sample_segment(
            self._h, int(i0), int(i1), shots, u.ctypes.data_as(_DP), uin,
            None if ein is None else ein.ctypes.data_as(_DP),
            None if nin is None else nin.ctypes.data_as(C.POINTER(N.I32)), C.byref(uo), eout.ctypes.data_as(_DP),
            nout.ctypes.data_as(C.POINTER(N.I32)), bits))
        raw = bits.raw.decode()
        return eout[: uo.value], nout, [raw[i * w:(i + 1) * w] for i in range(shots)]

    def sample_segment_dev(self, i0, i1, u, env_out, env_in=None, node_in=None):
        """sample_segment with the prefix environments in HBM: env_in
        (U x D_left) and env_out (capacity shots x D_right) are contiguous
        complex128 CUDA tensors on the state's device (the sharded sampler's
        NCCL hand-off buffers). Returns (U', node_out, bits); env_out[:U']
        holds the distinct prefixes' environments."""
        u = np.ascontiguousarray(u, dtype=np.float64)
        shots, w = u.shape
        if env_out.shape[0] < shots or env_out.shape[1] != int(self.bond_dims()[i1]) or not env_out.is_contiguous():
            raise ValueError("env_out must be a contiguous (shots x D_right) tensor")
        uin, nin = 1, None
        if env_in is not None:
            if not env_in.is_contiguous():
                raise ValueError("env_in must be contiguous")
            uin = int(env_in.shape[0])
            nin = np.ascontiguousarray(node_in, dtype=np.int32)
        nout = np.zeros(shots, dtype=np.int32)
        bits = C.create_string_buffer(shots * w)
        uo = N.I32()
        check(N.lib().mpsim_gpu_sample_segment_dev(
            self._h, int(i0), int(i1), shots, u.ctypes.data_as(_DP), uin,
            None if env_in is None else C.c_void_p(env_in.data_ptr()),
            None if nin is None else nin.ctypes.data_as(C.POINTER(N.I32)), C.byref(uo),
            C.c_void_p(env_out.data_ptr()), nout.ctypes.data_as(C.POINTER(N.I32)), bits))
        raw = bits.raw.decode()
        return uo.value, nout, [raw[i * w:(i + 1) * w] for i in range(shots)]

    # ---- environment forms (site-sharded chains, SURVEY 8(e) queries)
    def amplitudes_env(self, bitstrings, env_in=None, i0=0, i1=None) -> np.ndarray:
        """Row environments of bit strings (length n, sites [i0, i1) read)
        continued from env_in (count x D_left) -> count x D_right."""
        n = self.n
        i1 = n if i1 is None else int(i1)
        for b in bitstrings:
            if len(b) != n:
                raise ValueError(f"bit string length {len(b)} does not match qubit count {n}")
        dims = self.bond_dims()
        count = len(bitstrings)
        ein = None
        if env_in is not None:
            ein = np.ascontiguousarray(env_in, dtype=np.complex128).reshape(count, int(dims[i0]))
        out = np.zeros((count, int(dims[i1])), dtype=np.complex128)
        check(N.lib().mpsim_gpu_amplitudes_env(self._h, int(i0), i1, "".join(bitstrings).encode(), count,
                                               None if ein is None else ein.ctypes.data_as(_DP),
                                               out.ctypes.data_as(_DP)))
        return out

    def transfer_env(self, other: "MpsState", env_in=None, op=None, q=-1, i0=0, i1=None) -> np.ndarray:
        """E' = sum_p A_p^H E B_p over sites [i0, i1) of self (A) and other (B),
        op (2x2) applied to B at site q: D_left(A) x D_left(B) -> D_right(A) x D_right(B)."""
        i1 = self.n if i1 is None else int(i1)
        da, db = self.bond_dims(), other.bond_dims()
        ein = None
        if env_in is not None:
            ein = np.ascontiguousarray(env_in, dtype=np.complex128).reshape(int(da[i0]), int(db[i0]))
        o = None if op is None else _cm(op, 2)
        out = np.zeros((int(da[i1]), int(db[i1])), dtype=np.complex128)
        check(N.lib().mpsim_gpu_transfer_env(self._h, other._h, int(i0), i1,
                                             None if o is None else o.ctypes.data_as(_DP), int(q),
                                             None if ein is None else ein.ctypes.data_as(_DP),
                                             out.ctypes.data_as(_DP)))
        return out

    def to_statevector(self, max_qubits=20) -> np.ndarray:
        n = self.n
        if n > max_qubits:
            raise ValueError(f"statevector export capped at {max_qubits} qubits, got {n}")
        out = np.zeros(2 << n)
        check(N.lib().mpsim_gpu_to_statevector(self._h, int(max_qubits), out.ctypes.data_as(_DP)))
        return out.view(np.complex128)

    def move_center(self, c):
        check(N.lib().mpsim_gpu_move_center(self._h, int(c)))

    def left_canonicalize(self):
        self.move_center(self.n - 1)

    def right_canonicalize(self):
        self.move_center(0)

    def expect_1q(self, op, q) -> complex:
        op = _cm(op, 2)
        out = np.zeros(2)
        check(N.lib().mpsim_gpu_expect_1q(self._h, op.ctypes.data_as(_DP), int(q), out.ctypes.data_as(_DP)))
        return complex(out[0], out[1])

    def expect_2q(self, op_a, qa, op_b, qb) -> complex:
        a, b = _cm(op_a, 2), _cm(op_b, 2)
        out = np.zeros(2)
        check(N.lib().mpsim_gpu_expect_2q(self._h, a.ctypes.data_as(_DP), int(qa), b.ctypes.data_as(_DP), int(qb),
                                          out.ctypes.data_as(_DP)))
        return complex(out[0], out[1])

    # ---- instrumentation
    def counters(self):
        l, ms, sw = N.I64(), C.c_double(), N.I64()
        check(N.lib().mpsim_gpu_counters(self._h, C.byref(l), C.byref(ms), C.byref(sw)))
        jl, jms, sf, gf = N.I64(), C.c_double(), C.c_double(), C.c_double()
        check(N.lib().mpsim_gpu_kernel_counters(self._h, C.byref(jl), C.byref(jms), C.byref(sf), C.byref(gf)))
        h2d, d2h = N.I64(), N.I64()
        check(N.lib().mpsim_gpu_transfer_counters(self._h, C.byref(h2d), C.byref(d2h)))
        return dict(launches=l.value, device_ms=ms.value, sweeps=sw.value, jacobi_launches=jl.value,
                    jacobi_ms=jms.value, svd_flops=sf.value, gate_flops=gf.value, h2d_bytes=h2d.value,
                    d2h_bytes=d2h.value)

    def reset_counters(self):
        check(N.lib().mpsim_gpu_reset_counters(self._h))

    def synchronize(self):
        check(N.lib().mpsim_gpu_synchronize(self._h))


def execute(state: MpsState, gates, max_bond=None, cutoff=0.0, bondprop=False):
    """execute_serial semantics (executor.cpp:73-97) with layer-batched launches.

    ``gates`` is a fused gate list [(q0, q1, matrix)]. Returns a dict with the
    ExecStats fields and the per-gate reports (input order).
    """
    arr = make_gates(gates)
    reps = (N.Report * max(1, len(gates)))()
    st = N.ExecStats()
    p = _policy(max_bond, cutoff)
    check(N.lib().mpsim_gpu_execute(state._h, arr, len(gates), C.byref(p),
                                    N.NONLOCAL_BONDPROP if bondprop else N.NONLOCAL_SWAP, C.byref(st), reps))
    reps = list(reps)[: len(gates)]
    return dict(peak_bond=st.peak_bond, total_discarded_weight=st.total_discarded_weight, layers=st.layers,
                gates=st.gates, kernel_launches=st.kernel_launches, device_ms=st.device_ms,
                gate_w=np.array([r.discarded_weight for r in reps]),
                gate_k=np.array([r.new_bond for r in reps], dtype=np.int64),
                svd_count=np.array([r.svd_count for r in reps], dtype=np.int64))


# execute_parallel (executor.cpp:99-232): the GPU batches each layer into one
# launch sequence, so "workers" has no meaning beyond API compatibility.
def execute_parallel(state: MpsState, gates, max_bond=None, cutoff=0.0, workers=1):
    if workers < 1:
        raise ValueError("worker count must be >= 1")
    for q0, q1, _ in gates:
        if q1 is not None and q1 >= 0 and abs(q1 - q0) != 1:
            raise ValueError("parallel execution requires a local-gate plan")
    return execute(state, gates, max_bond, cutoff)


class Sampler:
    """Sampler (sampler.hpp:50-86)."""

    def __init__(self, state: MpsState, memoize=True, cache_cap=0):
        h = C.c_void_p()
        check(N.lib().mpsim_gpu_sampler_create(state._h, 1 if memoize else 0, int(cache_cap), C.byref(h)))
        self._h = h
        self._n = state.n

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and N._lib is not None:
            N._lib.mpsim_gpu_sampler_destroy(h)
            self._h = None

    def sample(self, shots, seed):
        u = N.I32()
        check(N.lib().mpsim_gpu_sample(self._h, int(shots), int(seed), C.byref(u)))
        out = {}
        buf = C.create_string_buffer(self._n + 1)
        cnt = N.U64()
        for i in range(u.value):
            check(N.lib().mpsim_gpu_sampler_result(self._h, i, buf, C.byref(cnt)))
            out[buf.raw[: self._n].decode()] = cnt.value
        return out

    def stats(self):
        h, s = N.U64(), N.U64()
        check(N.lib().mpsim_gpu_sampler_stats(self._h, C.byref(h), C.byref(s)))
        return h.value, s.value

    @property
    def cache_hits(self):
        return self.stats()[0]

    @property
    def cache_size(self):
        return self.stats()[1]

    def clear_cache(self):
        check(N.lib().mpsim_gpu_sampler_clear_cache(self._h))


def uniform_variates(seed, skip, count) -> np.ndarray:
    """std::mt19937_64(seed) draws skip .. skip + count as (x >> 11) 2^-53."""
    out = np.zeros(int(count))
    check(N.lib().mpsim_uniform_variates(int(seed), int(skip), int(count), out.ctypes.data_as(_DP)))
    return out


def sample(state: MpsState, shots, seed, memoize=True, cache_cap=0):
    return Sampler(state, memoize, cache_cap).sample(shots, seed)
