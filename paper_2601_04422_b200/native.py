"""ctypes binding of ``libmpsim_gpu.so`` (the C ABI in ``include/mpsim_gpu.h``).

There is no CPU fallback: importing this module on a machine without the
built library raises immediately, and every call that fails on the device
raises with the library's message.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmpsim_gpu.so")

MPSIM_OK, MPSIM_EINVAL, MPSIM_EPARSE, MPSIM_ENUMERIC, MPSIM_ELOGIC, MPSIM_ECUDA = 0, 1, 2, 3, 4, 5
UNBOUNDED = (1 << 63) - 1
NONLOCAL_SWAP, NONLOCAL_BONDPROP = 0, 1

I32, I64, U64, DBL = C.c_int32, C.c_int64, C.c_uint64, C.c_double
DP = C.POINTER(C.c_double)
VP = C.c_void_p


class Policy(C.Structure):
    _fields_ = [("max_bond", I64), ("cutoff", DBL)]


class Report(C.Structure):
    _fields_ = [("discarded_weight", DBL), ("new_bond", I64), ("svd_count", I32), ("reserved", I32)]

    def __repr__(self):
        return f"Report(w={self.discarded_weight}, k={self.new_bond}, svd={self.svd_count})"


class Gate(C.Structure):
    _fields_ = [("q0", I32), ("q1", I32), ("u", DBL * 32)]


class ExecStats(C.Structure):
    _fields_ = [("peak_bond", I64), ("total_discarded_weight", DBL), ("layers", I32), ("gates", I32),
                ("kernel_launches", I64), ("device_ms", DBL)]


class PrimOp(C.Structure):
    _fields_ = [("kind", I32), ("q0", I32), ("q1", I32), ("nparams", I32), ("params", DBL * 3)]


class CircuitInfo(C.Structure):
    _fields_ = [("n_qubits", I32), ("n_clbits", I32), ("has_measure_all", I32), ("n_ops", I32)]


class RunConfig(C.Structure):
    _fields_ = [("qasm_path", C.c_char_p), ("qasm_text", C.c_char_p), ("sidecar_path", C.c_char_p),
                ("sidecar_json", C.c_char_p), ("input_label", C.c_char_p), ("backend", I32), ("nonlocal_", I32),
                ("max_bond", I64), ("cutoff", DBL), ("shots", U64), ("seed", U64), ("workers", I32),
                ("memoize", I32), ("cache_cap", U64), ("statevector_cap", I32), ("device", I32),
                ("chi_hint", I64)]


class ParseError(ValueError):
    """mpsim::ParseError (errors.hpp:22-37): carries the 1-based line and column."""

    def __init__(self, msg, line=0, column=0):
        super().__init__(msg)
        self.line, self.column = line, column


class ConfigError(ValueError):
    """mpsim::ConfigError (errors.hpp:39-43)."""


class NumericError(RuntimeError):
    """mpsim::NumericError (errors.hpp:45-48)."""


class LogicError(RuntimeError):
    """std::logic_error (validate / span guard)."""


class DeviceError(RuntimeError):
    """CUDA runtime failure."""


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    sig = {
        "mpsim_gpu_last_error": (C.c_char_p, []),
        "mpsim_gpu_state_create": (C.c_int, [I32, I64, I32, C.POINTER(VP)]),
        "mpsim_gpu_state_destroy": (C.c_int, [VP]),
        "mpsim_gpu_state_copy": (C.c_int, [VP, C.POINTER(VP)]),
        "mpsim_gpu_num_qubits": (C.c_int, [VP, C.POINTER(I32)]),
        "mpsim_gpu_bond_dims": (C.c_int, [VP, C.POINTER(I64)]),
        "mpsim_gpu_chi_capacity": (C.c_int, [VP, C.POINTER(I64)]),
        "mpsim_gpu_ortho_center": (C.c_int, [VP, C.POINTER(I32)]),
        "mpsim_gpu_set_ortho_center": (C.c_int, [VP, I32]),
        "mpsim_gpu_set_bond_dim": (C.c_int, [VP, I32, I64]),
        "mpsim_gpu_validate": (C.c_int, [VP]),
        "mpsim_gpu_get_site": (C.c_int, [VP, I32, C.POINTER(I64), C.POINTER(I64), DP]),
        "mpsim_gpu_set_site": (C.c_int, [VP, I32, I64, I64, DP]),
        "mpsim_gpu_set_open_boundaries": (C.c_int, [VP, I32]),
        "mpsim_gpu_site_slot": (C.c_int, [VP, I32, C.POINTER(VP), C.POINTER(I64)]),
        "mpsim_gpu_set_site_dims": (C.c_int, [VP, I32, I64, I64]),
        "mpsim_gpu_apply_1q": (C.c_int, [VP, DP, I32, C.POINTER(Report)]),
        "mpsim_gpu_apply_2q": (C.c_int, [VP, DP, I32, I32, I32, C.POINTER(Policy), C.POINTER(Report)]),
        "mpsim_gpu_apply_layer": (C.c_int, [VP, C.POINTER(Gate), I32, C.POINTER(Policy), C.POINTER(Report)]),
        "mpsim_gpu_execute": (C.c_int, [VP, C.POINTER(Gate), I32, C.POINTER(Policy), I32, C.POINTER(ExecStats),
                                        C.POINTER(Report)]),
        "mpsim_gpu_svd": (C.c_int, [I32, I32, DP, I64, DBL, I32, C.POINTER(I64), DP, DP, DP, DP]),
        "mpsim_gpu_norm": (C.c_int, [VP, DP]),
        "mpsim_gpu_amplitudes": (C.c_int, [VP, C.c_char_p, I32, DP]),
        "mpsim_gpu_overlap": (C.c_int, [VP, VP, DP]),
        "mpsim_gpu_to_statevector": (C.c_int, [VP, I32, DP]),
        "mpsim_gpu_move_center": (C.c_int, [VP, I32]),
        "mpsim_gpu_sweep_left": (C.c_int, [VP, I32, I32]),
        "mpsim_gpu_sweep_right": (C.c_int, [VP, I32, I32]),
        "mpsim_gpu_site_norm2": (C.c_int, [VP, I32, DP]),
        "mpsim_gpu_amplitudes_env": (C.c_int, [VP, I32, I32, C.c_char_p, I32, DP, DP]),
        "mpsim_gpu_transfer_env": (C.c_int, [VP, VP, I32, I32, DP, I32, DP, DP]),
        "mpsim_gpu_expect_1q": (C.c_int, [VP, DP, I32, DP]),
        "mpsim_gpu_expect_2q": (C.c_int, [VP, DP, I32, DP, I32, DP]),
        "mpsim_gpu_sampler_create": (C.c_int, [VP, I32, U64, C.POINTER(VP)]),
        "mpsim_gpu_sampler_destroy": (C.c_int, [VP]),
        "mpsim_gpu_sample": (C.c_int, [VP, U64, U64, C.POINTER(I32)]),
        "mpsim_gpu_sampler_result": (C.c_int, [VP, I32, C.c_char_p, C.POINTER(U64)]),
        "mpsim_gpu_sampler_stats": (C.c_int, [VP, C.POINTER(U64), C.POINTER(U64)]),
        "mpsim_gpu_sampler_clear_cache": (C.c_int, [VP]),
        "mpsim_gpu_sample_segment": (C.c_int, [VP, I32, I32, U64, DP, I32, DP, C.POINTER(I32), C.POINTER(I32), DP,
                                               C.POINTER(I32), C.c_char_p]),
        "mpsim_gpu_sample_segment_dev": (C.c_int, [VP, I32, I32, U64, DP, I32, VP, C.POINTER(I32),
                                                   C.POINTER(I32), VP, C.POINTER(I32), C.c_char_p]),
        "mpsim_uniform_variates": (C.c_int, [U64, U64, U64, DP]),
        "mpsim_gpu_counters": (C.c_int, [VP, C.POINTER(I64), DP, C.POINTER(I64)]),
        "mpsim_gpu_kernel_counters": (C.c_int, [VP, C.POINTER(I64), DP, DP, DP]),
        "mpsim_gpu_transfer_counters": (C.c_int, [VP, C.POINTER(I64), C.POINTER(I64)]),
        "mpsim_gpu_reset_counters": (C.c_int, [VP]),
        "mpsim_gpu_synchronize": (C.c_int, [VP]),
        "mpsim_free": (None, [VP]),
        "mpsim_parse_qasm": (C.c_int, [C.c_char_p, C.POINTER(CircuitInfo), C.POINTER(PrimOp), I32]),
        "mpsim_last_parse_location": (C.c_int, [C.POINTER(I32), C.POINTER(I32)]),
        "mpsim_fuse_qasm": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(I32), C.POINTER(C.POINTER(Gate)),
                                      C.POINTER(C.POINTER(I32)), C.POINTER(I32)]),
        "mpsim_plan_layers": (C.c_int, [C.POINTER(Gate), I32, I32, C.POINTER(C.POINTER(Gate)),
                                        C.POINTER(C.POINTER(I32)), C.POINTER(I32), C.POINTER(I32)]),
        "mpsim_gen_ghz_qasm": (C.c_int, [I32, I32, C.POINTER(VP)]),
        "mpsim_gen_brickwork_qasm": (C.c_int, [I32, I32, U64, I32, I32, C.POINTER(VP), C.POINTER(VP)]),
        "mpsim_run_config_defaults": (None, [C.POINTER(RunConfig)]),
        "mpsim_gpu_run_circuit": (C.c_int, [C.POINTER(RunConfig), C.POINTER(VP)]),
        # multi-GPU shards (csrc/shard.cu)
        "mpsim_shard_bounds": (C.c_int, [I32, I32, I64, C.POINTER(I32)]),
        "mpsim_shard_partition_layer": (C.c_int, [C.POINTER(Gate), I32, I32, I32, I32, I32, C.POINTER(Gate),
                                                  C.POINTER(I32), C.POINTER(I32), C.POINTER(I32)]),
        "mpsim_gpu_nccl_unique_id": (C.c_int, [VP]),
        "mpsim_gpu_shard_create": (C.c_int, [I32, I64, I32, I32, VP, I32, C.POINTER(VP)]),
        "mpsim_gpu_shard_destroy": (C.c_int, [VP]),
        "mpsim_gpu_shard_info": (C.c_int, [VP, C.POINTER(I32), C.POINTER(I32), C.POINTER(VP)]),
        "mpsim_gpu_shard_set_site": (C.c_int, [VP, I32, I64, I64, DP]),
        "mpsim_gpu_shard_get_site": (C.c_int, [VP, I32, C.POINTER(I64), C.POINTER(I64), DP]),
        "mpsim_gpu_shard_bond_dims": (C.c_int, [VP, C.POINTER(I64)]),
        "mpsim_gpu_shard_apply_layer": (C.c_int, [VP, C.POINTER(Gate), I32, C.POINTER(Policy),
                                                  C.POINTER(ExecStats)]),
        "mpsim_gpu_shard_execute": (C.c_int, [VP, C.POINTER(Gate), I32, C.POINTER(Policy), C.POINTER(ExecStats)]),
        "mpsim_gpu_shard_amplitudes": (C.c_int, [VP, C.c_char_p, I32, DP]),
        "mpsim_gpu_shard_overlap": (C.c_int, [VP, VP, DP]),
        "mpsim_gpu_shard_norm": (C.c_int, [VP, DP]),
        "mpsim_gpu_shard_expect_1q": (C.c_int, [VP, DP, I32, DP]),
        "mpsim_gpu_shard_move_center": (C.c_int, [VP, I32]),
        "mpsim_gpu_shard_ortho_center": (C.c_int, [VP, C.POINTER(I32)]),
        "mpsim_gpu_shard_sample": (C.c_int, [VP, U64, U64, U64, C.POINTER(I32)]),
        "mpsim_gpu_shard_sample_result": (C.c_int, [VP, I32, C.c_char_p, C.POINTER(U64)]),
        "mpsim_gpu_shard_allreduce": (C.c_int, [VP, DP, I32, I32]),
        "mpsim_gpu_shard_barrier": (C.c_int, [VP]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def exported_symbols():
    """Names declared in include/mpsim_gpu.h (for the ABI-surface test)."""
    import re
    hdr = os.path.join(os.path.dirname(_HERE), "include", "mpsim_gpu.h")
    with open(hdr) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(mpsim_[a-z0-9_]+)\s*\(", text)))


def check(rc: int):
    if rc == MPSIM_OK:
        return
    msg = lib().mpsim_gpu_last_error().decode()
    if rc == MPSIM_EINVAL:
        raise ValueError(msg)
    if rc == MPSIM_EPARSE:
        line, col = I32(), I32()
        lib().mpsim_last_parse_location(C.byref(line), C.byref(col))
        raise ParseError(msg, line.value, col.value)
    if rc == MPSIM_ENUMERIC:
        raise NumericError(msg)
    if rc == MPSIM_ELOGIC:
        raise LogicError(msg)
    raise DeviceError(msg)
