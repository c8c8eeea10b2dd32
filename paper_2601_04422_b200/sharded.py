"""Contiguous site sharding of one MPS chain across GPUs.

A thin binding of the library's multi-GPU layer (csrc/shard.cu,
``mpsim_gpu_shard_*`` in include/mpsim_gpu.h): rank r owns sites [lo, hi)
with even, cost-weighted cut points plus a ghost slot; straddling gates of odd
brick layers exchange the boundary site over NCCL (send/recv on the shard's
stream, NVLink/NVSwitch); queries hand environments rank to rank; centre moves
and the sampler run the reference's steps in the reference's order. All data
movement and arithmetic is in libmpsim_gpu.so (C++/CUDA/NCCL); this module only
marshals arguments and bootstraps the NCCL communicator: rank 0's unique id
reaches the other ranks over a plain TCP socket (no torch).
"""
from __future__ import annotations

import ctypes as C
import os
import socket
import time

import numpy as np

from . import native as N
from .mps import MpsState, _policy, make_gates
from .native import check

_DP = N.DP


def _lib():
    return N.lib()  # signatures of the mpsim_gpu_shard_* entry points live in native.py


REDUCE_SUM, REDUCE_MAX, REDUCE_MIN = 0, 1, 2


def shard_bounds(n: int, world: int, chi: int | None = None):
    """Even-aligned contiguous ranges [b_r, b_{r+1}) (mpsim_shard_bounds):
    cost-weighted with a bond cap chi, an even split without."""
    out = (N.I32 * (world + 1))()
    check(_lib().mpsim_shard_bounds(int(n), int(world), 0 if chi is None else int(chi), out))
    return list(out)


def partition_layer(gates, lo, hi, rank, world):
    """One layer (global indices) for the shard [lo, hi)
    (mpsim_shard_partition_layer): the gates this rank applies as
    [(q0, q1, matrix)] in local indices (a gate on (hi-1, hi) uses the ghost
    slot), and whether it lends its first site left / borrows the right
    neighbour's."""
    arr = make_gates(gates)
    out = (N.Gate * max(1, len(gates)))()
    nl, sl, sr = N.I32(), N.I32(), N.I32()
    check(_lib().mpsim_shard_partition_layer(arr, len(gates), lo, hi, rank, world, out, C.byref(nl), C.byref(sl),
                                             C.byref(sr)))
    local = []
    for i in range(nl.value):
        g = out[i]
        dim = 2 if g.q1 < 0 else 4
        m = np.frombuffer(bytes(g.u), dtype=np.complex128)[: dim * dim].reshape(dim, dim).copy()
        local.append((g.q0, g.q1, m))
    return local, bool(sl.value), bool(sr.value)


def nccl_rendezvous(rank: int, world: int, addr: str | None = None, port: int | None = None, timeout=300.0):
    """Rank 0 draws the NCCL unique id and hands it to the other ranks over a
    TCP socket at MASTER_ADDR : MASTER_PORT + 1 (the launcher's own store keeps
    MASTER_PORT); returns the 128-byte id on every rank."""
    addr = addr or os.environ.get("MASTER_ADDR", "127.0.0.1")
    port = int(port or int(os.environ.get("MPSIM_RDZV_PORT", int(os.environ.get("MASTER_PORT", "29500")) + 1)))
    if rank == 0:
        buf = C.create_string_buffer(128)
        check(_lib().mpsim_gpu_nccl_unique_id(buf))
        uid = buf.raw
        with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as srv:
            srv.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
            srv.bind((addr, port))
            srv.listen(world)
            srv.settimeout(timeout)
            for _ in range(world - 1):
                c, _ = srv.accept()
                with c:
                    c.sendall(uid)
        return uid
    t0 = time.time()
    while True:
        try:
            with socket.create_connection((addr, port), timeout=10) as c:
                data = b""
                while len(data) < 128:
                    part = c.recv(128 - len(data))
                    if not part:
                        break
                    data += part
                if len(data) == 128:
                    return data
        except OSError:
            pass
        if time.time() - t0 > timeout:
            raise TimeoutError("NCCL id rendezvous timed out")
        time.sleep(0.2)


class ShardedChain:
    """One rank's shard of an n-qubit chain (mpsim_gpu_shard)."""

    def __init__(self, n, chi, rank=0, world=1, device=0, nccl_id=None):
        self.n, self.chi, self.rank, self.world, self.device = n, chi, rank, world, device
        os.environ.setdefault("NCCL_DEBUG", "WARN")  # no banner on stdout (bench.py prints one JSON line)
        if world > 1 and nccl_id is None:
            nccl_id = nccl_rendezvous(rank, world)
        h = C.c_void_p()
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        check(_lib().mpsim_gpu_shard_create(int(n), int(chi), int(rank), int(world), idbuf, int(device),
                                            C.byref(h)))
        self._h = h
        lo, hi, st = N.I32(), N.I32(), C.c_void_p()
        check(_lib().mpsim_gpu_shard_info(h, C.byref(lo), C.byref(hi), C.byref(st)))
        self.lo, self.hi = lo.value, hi.value
        self.state = MpsState(_handle=st)
        self.state._borrowed = True  # owned by the shard

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and N._lib is not None:
            if getattr(self, "state", None) is not None:
                self.state._h = None
            N._lib.mpsim_gpu_shard_destroy(h)
            self._h = None

    # ---- setup
    def set_site(self, i, t):
        t = np.ascontiguousarray(np.asarray(t, dtype=np.complex128))
        if t.ndim != 3 or t.shape[1] != 2:
            raise ValueError("site tensor must have shape (Dl, 2, Dr)")
        check(_lib().mpsim_gpu_shard_set_site(self._h, int(i), t.shape[0], t.shape[2], t.ctypes.data_as(_DP)))

    def site(self, i) -> np.ndarray:
        dl, dr = N.I64(), N.I64()
        check(_lib().mpsim_gpu_shard_get_site(self._h, int(i), C.byref(dl), C.byref(dr), None))
        out = np.zeros((dl.value, 2, dr.value), dtype=np.complex128)
        check(_lib().mpsim_gpu_shard_get_site(self._h, int(i), C.byref(dl), C.byref(dr), out.ctypes.data_as(_DP)))
        return out

    def finalize_setup(self):
        """Kept for callers of the earlier API: the ghost slot's extents now
        follow set_site of the last owned site."""

    # ---- plumbing
    def barrier(self):
        check(_lib().mpsim_gpu_shard_barrier(self._h))

    def allreduce(self, values, op=REDUCE_SUM):
        v = np.ascontiguousarray(np.asarray(values, dtype=np.float64).reshape(-1)).copy()
        check(_lib().mpsim_gpu_shard_allreduce(self._h, v.ctypes.data_as(_DP), len(v), int(op)))
        return v

    def max_over_ranks(self, x: float) -> float:
        return float(self.allreduce([x], REDUCE_MAX)[0])

    # ---- gates (global site indices)
    def apply_layer(self, gates, max_bond=None, cutoff=0.0):
        """One layer of disjoint local gates: exchange in, batched launch
        sequence, exchange out. device_ms spans all three."""
        arr = make_gates(gates)
        st = N.ExecStats()
        p = _policy(max_bond, cutoff)
        check(_lib().mpsim_gpu_shard_apply_layer(self._h, arr, len(gates), C.byref(p), C.byref(st)))
        return dict(device_ms=st.device_ms, peak_bond=st.peak_bond, total_discarded_weight=st.total_discarded_weight,
                    kernel_launches=st.kernel_launches)

    def execute(self, gates, max_bond=None, cutoff=0.0):
        """execute_parallel over the chain (non-local gates SWAP-lowered)."""
        arr = make_gates(gates)
        st = N.ExecStats()
        p = _policy(max_bond, cutoff)
        check(_lib().mpsim_gpu_shard_execute(self._h, arr, len(gates), C.byref(p), C.byref(st)))
        return dict(peak_bond=st.peak_bond, total_discarded_weight=st.total_discarded_weight, layers=st.layers,
                    gates=st.gates, kernel_launches=st.kernel_launches, device_ms=st.device_ms)

    # ---- queries over the whole chain
    def amplitudes(self, bitstrings):
        bits = "".join(bitstrings).encode()
        if len(bits) != len(bitstrings) * self.n:
            raise ValueError("bit strings must have n characters each")
        out = np.zeros(len(bitstrings), dtype=np.complex128)
        check(_lib().mpsim_gpu_shard_amplitudes(self._h, bits, len(bitstrings), out.ctypes.data_as(_DP)))
        return out

    def overlap(self, other: "ShardedChain") -> complex:
        out = np.zeros(2)
        check(_lib().mpsim_gpu_shard_overlap(self._h, other._h, out.ctypes.data_as(_DP)))
        return complex(out[0], out[1])

    def norm(self) -> float:
        out = C.c_double()
        check(_lib().mpsim_gpu_shard_norm(self._h, C.byref(out)))
        return out.value

    def expect_1q(self, op, q) -> complex:
        o = np.ascontiguousarray(np.asarray(op, dtype=np.complex128))
        if o.shape != (2, 2):
            raise ValueError("operator must be 2x2")
        out = np.zeros(2)
        check(_lib().mpsim_gpu_shard_expect_1q(self._h, o.ctypes.data_as(_DP), int(q), out.ctypes.data_as(_DP)))
        return complex(out[0], out[1])

    def move_center(self, c):
        check(_lib().mpsim_gpu_shard_move_center(self._h, int(c)))

    @property
    def ortho_center(self):
        v = N.I32()
        check(_lib().mpsim_gpu_shard_ortho_center(self._h, C.byref(v)))
        return None if v.value < 0 else v.value

    def sample(self, shots, seed, chunk=4096):
        """Ordered counts of `shots` perfect samples of the whole chain,
        identical to Sampler(state).sample(shots, seed) on one GPU."""
        u = N.I32()
        check(_lib().mpsim_gpu_shard_sample(self._h, int(shots), int(seed), int(chunk), C.byref(u)))
        out = {}
        buf = C.create_string_buffer(self.n + 1)
        cnt = N.U64()
        for i in range(u.value):
            check(_lib().mpsim_gpu_shard_sample_result(self._h, i, buf, C.byref(cnt)))
            out[buf.raw[: self.n].decode()] = cnt.value
        return out

    def bond_dims(self):
        """Bonds of the owned range [lo, hi]."""
        out = np.zeros(self.hi - self.lo + 1, dtype=np.int64)
        check(_lib().mpsim_gpu_shard_bond_dims(self._h, out.ctypes.data_as(C.POINTER(N.I64))))
        return out

    def counters(self):
        return self.state.counters()

    def reset_counters(self):
        self.state.reset_counters()
