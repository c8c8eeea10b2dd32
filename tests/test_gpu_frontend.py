"""run_circuit on the GPU: the reference pipeline tests
(tests/test_runner.cpp:37-168) plus counts / statistics parity with the
oracle's pipeline (parse -> fuse -> execute -> sample) on the same QASM."""
import json
import os

import numpy as np
import pytest

from paper_2601_04422_b200 import frontend as F
from tests.helpers import MT19937_64, gate_tuples

pytestmark = pytest.mark.gpu

# docs/run_output.schema.json, restated (the reference tree is not on the GPU box)
SCHEMA = {
    "type": "object",
    "required": ["config", "n_qubits", "peak_bond", "total_wall_ns", "total_discarded_weight", "layers"],
    "additionalProperties": False,
    "properties": {
        "config": {
            "type": "object",
            "required": ["input", "backend", "nonlocal", "max_bond", "cutoff", "shots", "seed", "workers",
                         "memoize"],
            "additionalProperties": False,
            "properties": {
                "input": {"type": "string"},
                "backend": {"type": "string", "enum": ["mps-serial", "mps-parallel", "statevector"]},
                "nonlocal": {"type": "string", "enum": ["swap", "bondprop"]},
                "max_bond": {"type": "integer", "minimum": 0},
                "cutoff": {"type": "number", "minimum": 0},
                "shots": {"type": "integer", "minimum": 0},
                "seed": {"type": "integer", "minimum": 0},
                "workers": {"type": "integer", "minimum": 1},
                "memoize": {"type": "boolean"},
            },
        },
        "n_qubits": {"type": "integer", "minimum": 1},
        "peak_bond": {"type": "integer", "minimum": 0},
        "total_wall_ns": {"type": "integer", "minimum": 0},
        "total_discarded_weight": {"type": "number", "minimum": 0},
        "layers": {"type": "array", "items": {
            "type": "object", "required": ["gates", "compute_ns", "sync_ns"], "additionalProperties": False,
            "properties": {"gates": {"type": "integer", "minimum": 0},
                           "compute_ns": {"type": "integer", "minimum": 0},
                           "sync_ns": {"type": "integer", "minimum": 0}}}},
        "counts": {"type": "object", "additionalProperties": {"type": "integer", "minimum": 0}},
    },
}


def violations(v, s, path="$"):
    """The draft-07 subset the schema uses (type, required, properties,
    additionalProperties, items, enum, minimum)."""
    out = []
    t = s.get("type")
    ok = {"object": isinstance(v, dict), "array": isinstance(v, list), "string": isinstance(v, str),
          "boolean": isinstance(v, bool), "integer": isinstance(v, int) and not isinstance(v, bool),
          "number": isinstance(v, (int, float)) and not isinstance(v, bool)}
    if t and not ok[t]:
        return [f"{path}: not {t}"]
    if "enum" in s and v not in s["enum"]:
        out.append(f"{path}: {v!r} not in enum")
    if "minimum" in s and v < s["minimum"]:
        out.append(f"{path}: below minimum")
    if t == "object":
        for k in s.get("required", []):
            if k not in v:
                out.append(f"{path}.{k}: missing")
        props = s.get("properties", {})
        extra = s.get("additionalProperties", True)
        for k, x in v.items():
            if k in props:
                out += violations(x, props[k], f"{path}.{k}")
            elif extra is False:
                out.append(f"{path}.{k}: not allowed")
            elif isinstance(extra, dict):
                out += violations(x, extra, f"{path}.{k}")
    if t == "array" and "items" in s:
        for i, x in enumerate(v):
            out += violations(x, s["items"], f"{path}[{i}]")
    return out


def test_ghz_counts_on_corner_strings(gpu):
    out = F.run_circuit(F.ghz_qasm(4), shots=1000, seed=5)
    assert out["n_qubits"] == 4 and out["peak_bond"] == 2
    assert set(out["counts"]) <= {"0000", "1111"} and sum(out["counts"].values()) == 1000


def test_shots_zero_omits_counts(gpu):
    out = F.run_circuit(F.ghz_qasm(4))
    assert "counts" not in out and len(out["layers"]) == 1
    assert out["layers"][0]["gates"] == 3  # h absorbed into the first cx


def test_identical_seeds_identical_counts(gpu):
    a = F.run_circuit(F.ghz_qasm(5), shots=2000, seed=77)
    b = F.run_circuit(F.ghz_qasm(5), shots=2000, seed=77)
    assert json.dumps(a["counts"]) == json.dumps(b["counts"])


def test_statevector_backend_sampling(gpu, oracle):
    """Backend::Statevector (runner.cpp:236-250): GHZ corner strings; and on a
    brickwork circuit the counts equal the reference's CDF sampler
    (runner.cpp:86-104) driven by mt19937_64 over the oracle statevector."""
    out = F.run_circuit(F.ghz_qasm(4), backend="statevector", shots=5000, seed=3)
    assert out["peak_bond"] == 0 and set(out["counts"]) <= {"0000", "1111"}
    n, shots, seed = 7, 3000, 19
    qasm, sc = F.brickwork_qasm(n, 3, 55, entangler="haar")
    got = F.run_circuit(qasm, sidecar_json=sc, backend="statevector", shots=shots, seed=seed)["counts"]
    psi = oracle.Circuit.brickwork(n, 3, 55, haar=True).statevector()
    cdf = np.cumsum(np.abs(psi) ** 2)
    e = MT19937_64(seed)
    want = {}
    for _ in range(shots):
        i = min(int(np.searchsorted(cdf, e.unit() * cdf[-1], side="right")), len(psi) - 1)
        b = format(i, f"0{n}b")
        want[b] = want.get(b, 0) + 1
    assert got == want


def test_parallel_agrees_with_serial(gpu):
    """test_runner.cpp:83-99 (brickwork n=6, depth 4, seed 10)."""
    qasm, _ = F.brickwork_qasm(6, 4, 10)
    a = F.run_circuit(qasm, shots=4000, seed=21)
    b = F.run_circuit(qasm, backend="mps-parallel", workers=3, shots=4000, seed=21)
    assert a["counts"] == b["counts"]
    assert len(b["layers"]) > 1
    assert sum(L["gates"] for L in b["layers"]) >= a["layers"][0]["gates"]


@pytest.mark.parametrize("backend", ["mps-serial", "mps-parallel"])
def test_counts_match_oracle_pipeline(gpu, oracle, backend):
    """The whole pipeline against the oracle's: same fused gates, same peak
    bond and discarded weight, identical counts from the perfect sampler."""
    n, depth, seed = 10, 6, 2601
    qasm, sc = F.brickwork_qasm(n, depth, seed, entangler="haar")
    out = F.run_circuit(qasm, sidecar_json=sc, backend=backend, cutoff=1e-12, shots=3000, seed=99)
    fused = oracle.Circuit.brickwork(n, depth, seed, haar=True).fuse()
    o = oracle.MpsState(n)
    ro = oracle.execute_serial(o, fused, None, 1e-12)
    assert out["peak_bond"] == ro["peak_bond"]
    assert abs(out["total_discarded_weight"] - ro["total_discarded_weight"]) <= 1e-22 + \
        1e-10 * ro["total_discarded_weight"]
    assert out["counts"] == oracle.Sampler(o).sample(3000, 99)


def test_capped_run_sampling_fails_like_the_reference(gpu, oracle):
    """A cap in a non-canonical gauge leaves the state unnormalised (P4: no
    centre move before gates); sampling then raises NumericError in both
    (sampler.cpp:36-40) and run_circuit exits with code 3."""
    n, depth, seed = 10, 6, 2601
    qasm, sc = F.brickwork_qasm(n, depth, seed, entangler="haar")
    with pytest.raises(F.NumericError, match="normalized") as ei:
        F.run_circuit(qasm, sidecar_json=sc, backend="mps-parallel", max_bond=8, cutoff=1e-12, shots=100)
    assert F.exit_code_for_error(ei.value) == 3
    o = oracle.MpsState(n)
    oracle.execute_serial(o, oracle.Circuit.brickwork(n, depth, seed, haar=True).fuse(), 8, 1e-12)
    with pytest.raises(oracle.NumericError):
        oracle.Sampler(o)
    rec = F.run_circuit(qasm, sidecar_json=sc, backend="mps-parallel", max_bond=8, cutoff=1e-12)
    assert rec["peak_bond"] == 8 and rec["total_discarded_weight"] > 0


def test_bondprop_serial_matches_oracle(gpu, oracle):
    """--nonlocal bondprop on the serial backend (runner.cpp:261-263)."""
    n = 8
    oc = oracle.Circuit.random(n, 50, 31, nonlocal_=True)
    qasm = "OPENQASM 2.0;\nqreg q[%d];\n" % n + "".join(
        f"{k}{'(' + ','.join('%.17g' % p for p in ps) + ')' if ps else ''} q[{a}]"
        + (f",q[{b}]" if b >= 0 else "") + ";\n" for k, a, b, ps in oc.ops())
    out = F.run_circuit(qasm, nonlocal_method="bondprop", cutoff=1e-12, shots=500, seed=4)
    o = oracle.MpsState(n)
    ro = oracle.execute_serial(o, oc.fuse(), None, 1e-12, bondprop=True)
    assert out["peak_bond"] == ro["peak_bond"]
    assert abs(out["total_discarded_weight"] - ro["total_discarded_weight"]) <= \
        1e-9 * max(ro["total_discarded_weight"], 1e-12)
    assert out["counts"] == oracle.Sampler(o).sample(500, 4)


def test_qasm_path_and_sidecar_pickup(gpu, tmp_path):
    """qasm_path reads the file; <path>.u4.json is picked up (runner.cpp:225-233)."""
    qasm, sc = F.brickwork_qasm(6, 2, 3, entangler="haar")
    p = tmp_path / "c.qasm"
    p.write_text(qasm)
    (tmp_path / "c.qasm.u4.json").write_text(sc)
    a = F.run_circuit(qasm_path=str(p), shots=300, seed=8)
    b = F.run_circuit(qasm, sidecar_json=sc, shots=300, seed=8)
    assert a["counts"] == b["counts"] and a["config"]["input"] == str(p)
    os.remove(tmp_path / "c.qasm.u4.json")
    c = F.run_circuit(qasm_path=str(p), shots=300, seed=8)  # plain u3 layers only
    assert c["peak_bond"] == 1


def test_run_output_schema(gpu):
    """test_runner.cpp:149-168: records validate; the checker sees violations."""
    rec = F.run_circuit(F.ghz_qasm(4), shots=100)
    assert violations(rec, SCHEMA) == []
    assert violations(F.run_circuit(F.ghz_qasm(4), backend="statevector"), SCHEMA) == []
    assert violations(F.run_circuit(F.ghz_qasm(4), backend="mps-parallel", workers=2), SCHEMA) == []
    broken = dict(rec)
    broken.pop("peak_bond")
    assert violations(broken, SCHEMA) != []
    assert rec["config"] == {"backend": "mps-serial", "cutoff": 0, "input": "<inline>", "max_bond": 0,
                             "memoize": True, "nonlocal": "swap", "seed": 1, "shots": 100, "workers": 1}


def test_statevector_cap(gpu):
    with pytest.raises(F.ConfigError, match="capped"):
        F.run_circuit(F.ghz_qasm(6), backend="statevector", statevector_cap=5)


def test_gate_tuples_roundtrip(gpu, oracle):
    """fuse_qasm output feeds the engine directly (execute == run_circuit)."""
    qasm, sc = F.brickwork_qasm(8, 4, 7, entangler="haar")
    n, g = F.fuse_qasm(qasm, sc)
    s = gpu.MpsState(n)
    r = gpu.execute(s, [x.as_tuple() for x in g], 4, 1e-12)
    o = oracle.MpsState(n)
    ro = oracle.execute_serial(o, oracle.Circuit.brickwork(8, 4, 7, haar=True).fuse(), 4, 1e-12)
    assert (r["gate_k"] == ro["gate_k"]).all()
    assert len(gate_tuples(oracle.Circuit.brickwork(8, 4, 7, haar=True).fuse())) == len(g)
