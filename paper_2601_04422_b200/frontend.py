"""Host front end of the reference pipeline over the C ABI:
``parse_qasm`` (qasm_parser.cpp), ``fuse_qasm`` (parse + inject_sidecar +
fuse_circuit, runner.cpp:168-190 / fusion.cpp:79-135), ``plan_layers``
(decompose_nonlocal + layerize, fusion.cpp:137-190), the generators
``ghz_qasm`` / ``brickwork_qasm`` (generators.cpp:52-145) and
``run_circuit`` (runner.cpp:219-289) returning the run record of
docs/run_output.schema.json (``run_output_to_json``, runner.cpp:291-328).

Errors follow the reference: ``ParseError`` (line, column), ``ConfigError``,
``NumericError``; ``exit_code_for_error`` maps them to 2 / 1 / 3
(runner.cpp:330-341). Parsing, fusion, planning and generation run on the
host inside libmpsim_gpu.so; run_circuit executes on the GPU.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field

import numpy as np

from . import native as N
from .native import ConfigError, NumericError, ParseError  # noqa: F401

GATE_NAMES = ["h", "x", "y", "z", "s", "sdg", "t", "tdg", "rx", "ry", "rz", "u1", "u2", "u3", "cx", "cz", "swap",
              "u4"]
BACKENDS = {"mps-serial": 0, "mps-parallel": 1, "statevector": 2}
NONLOCAL = {"swap": N.NONLOCAL_SWAP, "bondprop": N.NONLOCAL_BONDPROP}


def _check_cfg(rc):
    """ConfigError for MPSIM_EINVAL (runner.cpp's ConfigError / invalid_argument)."""
    try:
        N.check(rc)
    except ParseError:
        raise
    except ValueError as e:
        raise ConfigError(str(e)) from None


def _take_str(p: C.c_void_p) -> str | None:
    if not p.value:
        return None
    s = C.string_at(p.value).decode()
    N.lib().mpsim_free(p)
    return s


@dataclass
class PrimOp:
    """PrimOp (circuit.hpp:48-56); q1 = -1 for one-qubit ops."""
    kind: str
    q0: int
    q1: int
    params: list = field(default_factory=list)

    def two_qubit(self):
        return self.q1 >= 0


@dataclass
class Circuit:
    """Circuit (circuit.hpp:58-63)."""
    n_qubits: int
    n_clbits: int
    has_measure_all: bool
    ops: list


def parse_qasm(text: str) -> Circuit:
    L = N.lib()
    info = N.CircuitInfo()
    b = text.encode()
    N.check(L.mpsim_parse_qasm(b, C.byref(info), None, 0))
    ops = (N.PrimOp * max(1, info.n_ops))()
    N.check(L.mpsim_parse_qasm(b, C.byref(info), ops, info.n_ops))
    out = [PrimOp(GATE_NAMES[o.kind], o.q0, o.q1, list(o.params[: o.nparams])) for o in ops[: info.n_ops]]
    return Circuit(info.n_qubits, info.n_clbits, bool(info.has_measure_all), out)


@dataclass
class FusedGate:
    """FusedGate (circuit.hpp:71-81): q0 < q1, matrix in the (q0, q1) basis."""
    q0: int
    q1: int
    matrix: np.ndarray
    flipped: bool = False

    def two_qubit(self):
        return self.q1 >= 0

    def local(self):
        return not self.two_qubit() or self.q1 == self.q0 + 1

    def as_tuple(self):
        return (self.q0, self.q1, self.matrix)


def _gates_from(ptr, count, flipped=None):
    out = []
    for i in range(count):
        g = ptr[i]
        dim = 4 if g.q1 >= 0 else 2
        u = np.array(g.u[: 2 * dim * dim]).view(np.complex128).reshape(dim, dim).copy()
        out.append(FusedGate(g.q0, g.q1, u, bool(flipped[i]) if flipped else False))
    return out


def fuse_qasm(qasm: str, sidecar_json: str | None = None):
    """parse_qasm + inject_sidecar + fuse_circuit -> (n_qubits, [FusedGate])."""
    L = N.lib()
    n, cnt = N.I32(), N.I32()
    gp = C.POINTER(N.Gate)()
    fp = C.POINTER(N.I32)()
    _check_cfg(L.mpsim_fuse_qasm(qasm.encode(), sidecar_json.encode() if sidecar_json else None, C.byref(n),
                                 C.byref(gp), C.byref(fp), C.byref(cnt)))
    try:
        return n.value, _gates_from(gp, cnt.value, fp)
    finally:
        L.mpsim_free(C.cast(gp, C.c_void_p))
        L.mpsim_free(C.cast(fp, C.c_void_p))


def plan_layers(gates, n_qubits: int):
    """decompose_nonlocal + layerize -> list of layers of FusedGate."""
    from .mps import make_gates
    L = N.lib()
    tup = [g.as_tuple() if isinstance(g, FusedGate) else g for g in gates]
    arr = make_gates(tup)
    gp = C.POINTER(N.Gate)()
    lp = C.POINTER(N.I32)()
    cnt, nl = N.I32(), N.I32()
    N.check(L.mpsim_plan_layers(arr, len(tup), int(n_qubits), C.byref(gp), C.byref(lp), C.byref(cnt),
                                C.byref(nl)))
    try:
        flat = _gates_from(gp, cnt.value)
        layers = [[] for _ in range(nl.value)]
        for i, g in enumerate(flat):
            layers[lp[i]].append(g)
        return layers
    finally:
        L.mpsim_free(C.cast(gp, C.c_void_p))
        L.mpsim_free(C.cast(lp, C.c_void_p))


def ghz_qasm(n_qubits: int, measure: bool = False) -> str:
    p = C.c_void_p()
    _check_cfg(N.lib().mpsim_gen_ghz_qasm(int(n_qubits), int(measure), C.byref(p)))
    return _take_str(p)


def brickwork_qasm(n_qubits: int, depth: int, seed: int = 1, measure: bool = False, entangler: str = "cx"):
    """(qasm, sidecar_json or None); entangler "cx" or "haar" (generators.hpp:40-48)."""
    if entangler not in ("cx", "haar"):
        raise ConfigError(f"unknown entangler '{entangler}'")
    q, s = C.c_void_p(), C.c_void_p()
    _check_cfg(N.lib().mpsim_gen_brickwork_qasm(int(n_qubits), int(depth), int(seed), int(measure),
                                                int(entangler == "haar"), C.byref(q), C.byref(s)))
    return _take_str(q), _take_str(s)


def run_circuit(qasm_text: str | None = None, *, qasm_path: str | None = None, sidecar_path: str | None = None,
                sidecar_json: str | None = None, input_label: str | None = None, backend: str = "mps-serial",
                nonlocal_method: str = "swap", max_bond: int = 0, cutoff: float = 0.0, shots: int = 0,
                seed: int = 1, workers: int = 1, memoize: bool = True, cache_cap: int = 0,
                statevector_cap: int = 20, device: int = 0, chi_hint: int = 16) -> dict:
    """run_circuit + run_output_to_json (RunConfig fields, runner.hpp:46-62)."""
    if backend not in BACKENDS:
        raise ConfigError(f"unknown backend '{backend}'")
    if nonlocal_method not in NONLOCAL:
        raise ConfigError(f"unknown nonlocal method '{nonlocal_method}'")
    L = N.lib()
    cfg = N.RunConfig()
    L.mpsim_run_config_defaults(C.byref(cfg))
    enc = lambda s: s.encode() if s else None  # noqa: E731
    cfg.qasm_text, cfg.qasm_path = enc(qasm_text), enc(qasm_path)
    cfg.sidecar_path, cfg.sidecar_json, cfg.input_label = enc(sidecar_path), enc(sidecar_json), enc(input_label)
    cfg.backend, cfg.nonlocal_ = BACKENDS[backend], NONLOCAL[nonlocal_method]
    cfg.max_bond, cfg.cutoff, cfg.shots, cfg.seed = int(max_bond), float(cutoff), int(shots), int(seed)
    cfg.workers, cfg.memoize, cfg.cache_cap = int(workers), int(bool(memoize)), int(cache_cap)
    cfg.statevector_cap, cfg.device, cfg.chi_hint = int(statevector_cap), int(device), int(chi_hint)
    out = C.c_void_p()
    _check_cfg(L.mpsim_gpu_run_circuit(C.byref(cfg), C.byref(out)))
    return json.loads(_take_str(out))


def exit_code_for_error(e: BaseException) -> int:
    """runner.cpp:330-341: ConfigError 1, ParseError 2, NumericError 3, other 1."""
    if isinstance(e, ParseError):
        return 2
    if isinstance(e, NumericError):
        return 3
    return 1
