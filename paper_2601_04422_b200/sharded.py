"""Contiguous site sharding of one MPS chain across GPUs.

Rank r owns sites [lo, hi) with even boundaries, so even brick layers never
straddle a shard and odd layers straddle at exactly world-1 gates. A shard
that is not the last keeps one extra "ghost" slot after its last site. For a
layer with a gate on (hi-1, hi):
  1. rank r+1 sends its first site (a whole padded slot, NCCL send/recv over
     NVLink) and its extents to rank r, which records it in the ghost slot;
  2. every rank applies its own gates (the straddling one included on rank r)
     as one batched launch sequence;
  3. rank r sends the updated ghost site (k, 2, Dr) back; rank r+1 stores it
     as its first site, whose left bond is now k.
Gates are disjoint within a layer, so this reproduces the single-GPU result
gate for gate: the per-gate inputs never change with the shard count.
torch.distributed is only plumbing here: it carries the slot bytes; all the
arithmetic runs in libmpsim_gpu.so.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import native as N
from .mps import MpsState, execute


def shard_bounds(n: int, world: int, chi: int | None = None):
    """Even-aligned contiguous ranges [b_r, b_{r+1}). With a bond cap `chi`
    the cut points split the steady-state gate cost (the theta merge and SVD of
    the gate on (q, q+1) scale as D_q D_{q+1} D_{q+2}, bonds min(chi, 2^q,
    2^(n-q))) into equal parts, so the cheap edge gates do not leave the edge
    shards idle; without it the sites are split evenly."""
    if chi is None or world == 1:
        cum = [float(q) for q in range(n + 1)]
    else:
        bond = [min(chi, 2 ** min(q, n - q, 60)) for q in range(n + 1)]
        cost = [float(bond[q] * bond[q + 1] * bond[min(q + 2, n)]) for q in range(n)]
        cum = [0.0]
        for c in cost:
            cum.append(cum[-1] + c)
    b = [0]
    for r in range(1, world):
        target = r * cum[-1] / world
        x = min(range(n + 1), key=lambda q: abs(cum[q] - target))
        x -= x % 2
        x = max(b[-1] + 2, x)
        x = min(x, n - 2 * (world - r))  # leave room for the remaining shards
        b.append(x)
    b.append(n)
    return b


def partition_layer(gates, lo, hi, rank, world):
    """Split one layer (global indices) for the shard [lo, hi): the gates this
    rank applies (local indices; a gate on (hi-1, hi) uses the ghost slot) and
    whether it lends its first site left / borrows the right neighbour's."""
    local = []
    straddle_left = straddle_right = False
    for (q0, q1, u) in gates:
        if q1 is None or q1 < 0:
            if lo <= q0 < hi:
                local.append((q0 - lo, -1, u))
            continue
        a, b = min(q0, q1), max(q0, q1)
        if b != a + 1:
            raise ValueError("sharded layers take local gates (lower non-local gates to SWAP chains first)")
        if lo <= a and b < hi:
            local.append((q0 - lo, q1 - lo, u))
        elif rank < world - 1 and a == hi - 1:
            local.append((q0 - lo, q1 - lo, u))
            straddle_right = True
        elif rank > 0 and b == lo:
            straddle_left = True
    return local, straddle_left, straddle_right


class _CudaArray:
    """__cuda_array_interface__ view of a device slot, for torch.as_tensor."""

    def __init__(self, ptr, nelem):
        self.__cuda_array_interface__ = {"shape": (nelem,), "typestr": "<c16", "data": (ptr, False),
                                         "version": 3, "strides": None}


class ShardedChain:
    def __init__(self, n, chi, rank=0, world=1, device=0, dist=None):
        self.n, self.chi, self.rank, self.world, self.dist = n, chi, rank, world, dist
        b = shard_bounds(n, world, chi)
        self.lo, self.hi = b[rank], b[rank + 1]
        self.has_right = rank < world - 1
        self.n_local = self.hi - self.lo + (1 if self.has_right else 0)
        self.state = MpsState(self.n_local, chi_hint=chi, device=device)
        if world > 1:
            self.state.set_open_boundaries(True)
        self.device = device
        self._torch = None
        if world > 1:
            import torch
            self._torch = torch

    # ---- setup
    def set_site(self, i, t):
        assert self.lo <= i < self.hi
        self.state.set_site(i - self.lo, t)

    def finalize_setup(self):
        """Give the ghost slot extents consistent with the last owned bond."""
        if self.has_right:
            b = self.state.bond_dims()
            self.state.set_site_dims(self.n_local - 1, int(b[self.hi - self.lo]), 1)

    # ---- plumbing
    def _slot_tensor(self, local_i):
        ptr, chi = self.state.site_slot(local_i)
        return self._torch.as_tensor(_CudaArray(ptr, chi * 2 * chi), device=f"cuda:{self.device}")

    def barrier(self):
        if self.world > 1:
            self._torch.cuda.synchronize()
            self.dist.barrier()
        self.state.synchronize()

    def max_over_ranks(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self._torch.tensor([x], dtype=self._torch.float64, device=f"cuda:{self.device}")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def _exchange_in(self, straddle_left, straddle_right):
        """Step 1: ghost <- first site of the right neighbour."""
        torch, dist = self._torch, self.dist
        ops = []
        if straddle_left:  # my first site goes to rank-1
            b = self.state.bond_dims()
            dims = torch.tensor([b[0], b[1]], dtype=torch.int64, device=f"cuda:{self.device}")
            ops += [dist.P2POp(dist.isend, dims, self.rank - 1), dist.P2POp(dist.isend, self._slot_tensor(0),
                                                                          self.rank - 1)]
        if straddle_right:
            self._dims_in = torch.zeros(2, dtype=torch.int64, device=f"cuda:{self.device}")
            ops += [dist.P2POp(dist.irecv, self._dims_in, self.rank + 1),
                    dist.P2POp(dist.irecv, self._slot_tensor(self.n_local - 1), self.rank + 1)]
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
            torch.cuda.synchronize()
        if straddle_right:
            dl, dr = (int(x) for x in self._dims_in.tolist())
            self.state.set_site_dims(self.n_local - 1, dl, dr)

    def _exchange_out(self, straddle_left, straddle_right):
        """Step 3: updated ghost -> first site of the right neighbour."""
        torch, dist = self._torch, self.dist
        ops = []
        if straddle_right:
            b = self.state.bond_dims()
            dims = torch.tensor([b[-2], b[-1]], dtype=torch.int64, device=f"cuda:{self.device}")
            ops += [dist.P2POp(dist.isend, dims, self.rank + 1),
                    dist.P2POp(dist.isend, self._slot_tensor(self.n_local - 1), self.rank + 1)]
        if straddle_left:
            dims_in = torch.zeros(2, dtype=torch.int64, device=f"cuda:{self.device}")
            ops += [dist.P2POp(dist.irecv, dims_in, self.rank - 1),
                    dist.P2POp(dist.irecv, self._slot_tensor(0), self.rank - 1)]
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
            torch.cuda.synchronize()
        if straddle_left:
            dl, dr = (int(x) for x in dims_in.tolist())
            self.state.set_site_dims(0, dl, dr)

    # ---- one layer of disjoint gates in global site indices
    def apply_layer(self, gates, max_bond=None, cutoff=0.0):
        local, straddle_left, straddle_right = partition_layer(gates, self.lo, self.hi, self.rank, self.world)
        if self.world > 1:
            self._exchange_in(straddle_left, straddle_right)
        st = execute(self.state, local, max_bond, cutoff) if local else dict(device_ms=0.0)
        if self.world > 1:
            self._exchange_out(straddle_left, straddle_right)
        return st

    # ---- queries over the shards: the chain is sequential, so
    # each rank continues its left neighbour's environment over its owned
    # sites [lo, hi) and sends its own to the right; the last rank holds the
    # result and broadcasts it. NCCL moves the environments (count x chi or
    # chi x chi complex128) as device tensors.
    def _env_chain(self, compute, shape_in, result_len):
        """compute(env_in) on every rank in chain order (rank r receives the
        environment of rank r - 1); the last rank's result, flattened to
        result_len values, is returned on every rank."""
        torch, dist = self._torch, self.dist
        dev = f"cuda:{self.device}"
        env = None
        if self.rank > 0:
            t = torch.empty(shape_in, dtype=torch.complex128, device=dev)
            dist.recv(t, self.rank - 1)
            env = t.cpu().numpy()
        out = compute(env)
        if self.rank < self.world - 1:
            dist.send(torch.from_numpy(np.ascontiguousarray(out)).to(dev), self.rank + 1)
            res = torch.empty((result_len,), dtype=torch.complex128, device=dev)
        else:
            res = torch.from_numpy(np.ascontiguousarray(out.reshape(-1))).to(dev)
        dist.broadcast(res, self.world - 1)
        return res.cpu().numpy()

    def amplitudes(self, bitstrings):
        """amplitude (mps.cpp:204-221) of full-length bit strings of the chain."""
        k = self.hi - self.lo
        local = [b[self.lo:self.hi] + "0" * (self.state.n - k) for b in bitstrings]
        if self.world == 1:
            return self.state.amplitudes_env(local, None, 0, k)[:, 0]
        d0 = int(self.state.bond_dims()[0])
        return self._env_chain(lambda e: self.state.amplitudes_env(local, e, 0, k), (len(bitstrings), d0),
                               len(bitstrings))

    def _transfer(self, other, op=None, q=-1):
        k = self.hi - self.lo
        if self.world == 1:
            return complex(self.state.transfer_env(other.state, None, op, q, 0, k)[0, 0])
        da, db = int(self.state.bond_dims()[0]), int(other.state.bond_dims()[0])
        return complex(self._env_chain(lambda e: self.state.transfer_env(other.state, e, op, q, 0, k), (da, db), 1)[0])

    # ---- centre moves across the shards (move_center, mps.cpp:177-187): the
    # left sweep runs rank by rank towards the centre, each rank absorbing its
    # last R into its ghost copy of the right neighbour's first site and
    # handing it back; the right sweep mirrors it from the chain's end, the
    # left rank running the boundary step on its ghost slot. Same QRs in the
    # same order as MpsState.move_center.
    def _p2p(self, send=None, recv=None):
        torch, dist = self._torch, self.dist
        dev = f"cuda:{self.device}"
        ops = []
        if send is not None:
            li, dst = send
            b = self.state.bond_dims()
            dims = torch.tensor([b[li], b[li + 1]], dtype=torch.int64, device=dev)
            ops += [dist.P2POp(dist.isend, dims, dst), dist.P2POp(dist.isend, self._slot_tensor(li), dst)]
        if recv is not None:
            li, src = recv
            dims_in = torch.zeros(2, dtype=torch.int64, device=dev)
            ops += [dist.P2POp(dist.irecv, dims_in, src), dist.P2POp(dist.irecv, self._slot_tensor(li), src)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        torch.cuda.synchronize()
        if recv is not None:
            dl, dr = (int(x) for x in dims_in.tolist())
            self.state.set_site_dims(recv[0], dl, dr)

    def move_center(self, c):
        if not 0 <= c < self.n:
            raise ValueError("center out of range")
        if self.world == 1:
            self.state.move_center(c)
            return
        self.state.synchronize()
        bounds = shard_bounds(self.n, self.world, self.chi)
        rc = max(r for r in range(self.world) if bounds[r] <= c)
        k, ghost, r = self.hi - self.lo, self.hi - self.lo, self.rank
        if r <= rc:  # left sweep, ranks 0 .. rc in order
            if r > 0:
                self._p2p(send=(0, r - 1))   # my first site becomes r-1's ghost ...
                self._p2p(recv=(0, r - 1))   # ... and comes back with its R absorbed
            if r < rc:
                self._p2p(recv=(ghost, r + 1))
                self.state.sweep_left(0, k)
                self._p2p(send=(ghost, r + 1))
            else:
                self.state.sweep_left(0, c - self.lo)
        if r >= rc:  # right sweep, ranks world-1 .. rc in order
            if r < self.world - 1:
                self._p2p(recv=(ghost, r + 1))
                self.state.sweep_right(ghost, ghost)
                self._p2p(send=(ghost, r + 1))
            lo_step = 1 if r > rc else c - self.lo + 1
            if k - 1 >= lo_step:
                self.state.sweep_right(lo_step, k - 1)
            if r > rc:
                self._p2p(send=(0, r - 1))
                self._p2p(recv=(0, r - 1))
        bad = self._torch.zeros(1, dtype=self._torch.float64, device=f"cuda:{self.device}")
        if r == rc and np.sqrt(self.state.site_norm2(c - self.lo)) < 1e-14:
            bad += 1.0
        self.dist.all_reduce(bad)
        if bad.item() > 0:
            raise N.NumericError("cannot canonicalize a zero-norm state")
        self.center = c

    # ---- perfect sampling across the shards (Sampler, sampler.cpp:35-143)
    def _clone(self):
        c = object.__new__(ShardedChain)
        c.__dict__.update(self.__dict__)
        c.state = self.state.copy()
        if self.world > 1:
            c.state.set_open_boundaries(True)
        return c

    def sample(self, shots, seed, chunk=4096):
        """Counts of `shots` perfect samples, identical to Sampler(state).sample
        on the whole chain: a left + right canonicalised copy, then each rank
        walks its sites for every shot from the distinct-prefix environments
        its left neighbour hands over; variates are the reference's
        shot-major mt19937_64 stream restricted to the rank's sites."""
        from .mps import uniform_variates
        if shots <= 0:
            raise ValueError("shots must be positive")
        nrm = self.norm()
        if abs(nrm - 1.0) > 1e-8:  # sampler.cpp:36-40
            raise N.NumericError(f"sampling requires a normalized state, norm is {nrm:.6f}")
        prep = self._clone()
        prep.move_center(self.n - 1)  # left_canonicalize (sampler.cpp:46)
        prep.move_center(0)           # right_canonicalize (sampler.cpp:47)
        k, n = self.hi - self.lo, self.n
        counts, mine = {}, []
        torch, dist = self._torch, self.dist
        dev = f"cuda:{self.device}"
        dims = prep.state.bond_dims()
        d0, dk = int(dims[0]), int(dims[k])
        for c0 in range(0, shots, chunk):
            cs = min(chunk, shots - c0)
            u = uniform_variates(seed, c0 * n, cs * n).reshape(cs, n)[:, self.lo:self.hi]
            env_in = node_in = None
            if self.rank > 0:
                meta = torch.zeros(1, dtype=torch.int64, device=dev)
                dist.recv(meta, self.rank - 1)
                U = int(meta.item())
                env_in = torch.empty((U, d0), dtype=torch.complex128, device=dev)
                t_node = torch.empty((cs,), dtype=torch.int32, device=dev)
                dist.recv(env_in, self.rank - 1)
                dist.recv(t_node, self.rank - 1)
                node_in = t_node.cpu().numpy()   # synchronises: env_in is in place
            if self.world == 1:
                _, _, bits = prep.state.sample_segment(0, k, u)
                mine.extend(bits)
                continue
            env_out = torch.empty((cs, dk), dtype=torch.complex128, device=dev)
            U_out, node_out, bits = prep.state.sample_segment_dev(0, k, u, env_out, env_in, node_in)
            if self.rank < self.world - 1:
                # the prefix environments go from HBM to HBM, no host staging
                dist.send(torch.tensor([U_out], dtype=torch.int64, device=dev), self.rank + 1)
                dist.send(env_out[:U_out], self.rank + 1)
                dist.send(torch.from_numpy(node_out).to(dev), self.rank + 1)
            mine.extend(bits)
        # one gather after the chunk loop: no per-chunk collective, so rank r
        # runs chunk j while rank r + 1 is still on chunk j - 1 (the handed
        # environments are the only coupling between ranks)
        parts = [None] * self.world if self.world > 1 else [mine]
        if self.world > 1:
            dist.all_gather_object(parts, mine)
        for sh in range(shots):
            key = "".join(p[sh] for p in parts)
            counts[key] = counts.get(key, 0) + 1
        return dict(sorted(counts.items()))

    def overlap(self, other: "ShardedChain") -> complex:
        """<self|other> (mps.cpp:223-239) of two chains sharded alike."""
        return self._transfer(other)

    def norm(self) -> float:
        """mps.cpp:189-202."""
        return float(np.sqrt(max(self._transfer(self).real, 0.0)))

    def expect_1q(self, op, q) -> complex:
        """<psi|O_q|psi>, the P9 definition, with O applied on the owning shard."""
        own = self.lo <= q < self.hi
        return self._transfer(self, op if own else None, q - self.lo if own else -1)

    def bond_dims(self):
        """Bonds of the owned range [lo, hi]."""
        return self.state.bond_dims()[: self.hi - self.lo + 1]

    def counters(self):
        return self.state.counters()

    def reset_counters(self):
        self.state.reset_counters()
