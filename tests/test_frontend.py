"""Host front end on CPU: the product's QASM parser, fusion,
SWAP lowering / layering and generators inside libmpsim_gpu.so, checked
against the reference's own parser/fusion tests (tests/test_circuit.cpp,
tests/test_runner.cpp) and against the oracle's fusion (oracle/, which
restates fusion.cpp). Nothing here touches a GPU."""
import json

import numpy as np
import pytest

from paper_2601_04422_b200 import frontend as F
from tests.helpers import dense_apply_1q, dense_apply_2q, max_dev

HDR = 'OPENQASM 2.0;\ninclude "qelib1.inc";\n'


def qasm_of(ops, n):
    """An oracle op list as QASM text (angles at %.17g round-trip exactly)."""
    lines = [HDR + f"qreg q[{n}];"]
    for kind, q0, q1, params in ops:
        p = "(" + ",".join("%.17g" % x for x in params) + ")" if params else ""
        args = f"q[{q0}]" + (f",q[{q1}]" if q1 >= 0 else "")
        lines.append(f"{kind}{p} {args};")
    return "\n".join(lines) + "\n"


def sv_of(n, gates):
    psi = np.zeros(1 << n, dtype=complex)
    psi[0] = 1
    for g in gates:
        psi = dense_apply_2q(psi, g.matrix, g.q0, g.q1, n) if g.q1 >= 0 else dense_apply_1q(psi, g.matrix, g.q0, n)
    return psi


# ------------------------------------------------------------------ parser
# tests/test_circuit.cpp:46-137

def test_parser_direct_mapping():
    c = F.parse_qasm(HDR + "qreg q[2];\nh q[0];\ncx q[0],q[1];\n")
    assert c.n_qubits == 2 and len(c.ops) == 2
    assert (c.ops[0].kind, c.ops[0].q0) == ("h", 0)
    assert (c.ops[1].kind, c.ops[1].q0, c.ops[1].q1) == ("cx", 0, 1)
    assert not c.has_measure_all


def test_parser_parameter_expressions():
    c = F.parse_qasm("OPENQASM 2.0; qreg q[1];\nrz(pi/2) q[0];\nrx(-pi/4) q[0];\n"
                     "u3(2*pi/3, 0.5, 1e-3) q[0];\nu1((pi+1)/2) q[0];\nry(3*(1-2)) q[0];\n")
    p = [o.params for o in c.ops]
    assert abs(p[0][0] - np.pi / 2) <= 1e-15
    assert abs(p[1][0] + np.pi / 4) <= 1e-15
    assert abs(p[2][0] - 2 * np.pi / 3) <= 1e-15 and p[2][1] == 0.5 and abs(p[2][2] - 1e-3) <= 1e-18
    assert abs(p[3][0] - (np.pi + 1) / 2) <= 1e-15
    assert p[4][0] == -3.0


def test_parser_ghz64_roundtrip():
    c = F.parse_qasm(F.ghz_qasm(64))
    assert c.n_qubits == 64 and len(c.ops) == 64
    assert c.ops[0].kind == "h" and all(o.kind == "cx" for o in c.ops[1:])


def test_parser_measures_and_barriers():
    c = F.parse_qasm("OPENQASM 2.0; qreg q[2]; creg c[2];\nh q[0];\nbarrier q;\nbarrier q[0], q[1];\n"
                     "measure q[0] -> c[0];\nmeasure q[1] -> c[1];\n")
    assert c.n_clbits == 2 and len(c.ops) == 1 and c.has_measure_all
    assert F.parse_qasm("OPENQASM 2.0; qreg q[3]; creg c[3]; measure q -> c;").has_measure_all
    assert not F.parse_qasm("OPENQASM 2.0; qreg q[3]; creg c[3]; measure q[0] -> c[0];").has_measure_all


@pytest.mark.parametrize("text,line,fragment", [
    ("OPENQASM 2.0; qreg q[2];\nccx q[0],q[1];", 2, "unsupported gate"),
    ("OPENQASM 2.0; qreg q[2];\nh q[5];", 2, "out of range"),
    ("OPENQASM 2.0; qreg q[2];\nqreg r[2];", 2, "multiple qregs"),
    ("OPENQASM 2.0; qreg q[2];\nh q[0]", 2, "expected ';'"),
    ("OPENQASM 3.0; qreg q[1];", 1, "unsupported OPENQASM version"),
    ("OPENQASM 2.0; qreg q[2];\ncx q[1],q[1];", 2, "distinct"),
    ("OPENQASM 2.0; qreg q[1];\ngate foo a { }", 2, "unsupported statement"),
    ("OPENQASM 2.0; qreg q[1];\ninclude \"other.inc\";", 2, "unsupported include"),
    ("OPENQASM 2.0; qreg q[1];\nrz(1/0) q[0];", 2, "division by zero"),
    ("OPENQASM 2.0; qreg q[1];\nh(0.5) q[0];", 2, "takes no parameters"),
    ("OPENQASM 2.0; qreg q[1];\nu3(1,2) q[0];", 2, "expects 3 parameter"),
    ("OPENQASM 2.0;\nh q[0];", 2, "gate before qreg"),
    ("OPENQASM 2.0; qreg q[1];\nh r[0];", 2, "unknown register"),
    ("OPENQASM 2.0;", 1, "no qreg declared"),
])
def test_parser_errors_carry_line_and_column(text, line, fragment):
    with pytest.raises(F.ParseError) as ei:
        F.parse_qasm(text)
    assert ei.value.line == line, str(ei.value)
    assert fragment in str(ei.value)
    assert str(ei.value).startswith(f"line {line}, column ")


def test_parser_error_column():
    with pytest.raises(F.ParseError) as ei:
        F.parse_qasm("OPENQASM 2.0;\nqreg q[2];\nh q[0]; h nope[0];")
    assert ei.value.line == 3 and ei.value.column > 1


# ------------------------------------------------------------------ fusion
# tests/test_circuit.cpp:139-199

def test_fusion_h_twice_is_identity():
    n, g = F.fuse_qasm("OPENQASM 2.0; qreg q[1]; h q[0]; h q[0];")
    assert len(g) == 1 and g[0].q1 < 0
    assert np.abs(g[0].matrix - np.eye(2)).max() <= 1e-12


def test_fusion_1q_absorbed_into_following_cx():
    n, g = F.fuse_qasm("OPENQASM 2.0; qreg q[2]; h q[0]; cx q[0],q[1];")
    assert len(g) == 1 and (g[0].q0, g[0].q1) == (0, 1)
    h = np.array([[1, 1], [1, -1]]) / np.sqrt(2)
    cx = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]])
    assert np.abs(g[0].matrix - cx @ np.kron(h, np.eye(2))).max() <= 1e-12


def test_fusion_absorption_blocked_by_intervening_gate():
    text = "OPENQASM 2.0; qreg q[3]; cx q[0],q[1]; cx q[1],q[2]; h q[0];"
    n, g = F.fuse_qasm(text)
    assert len(g) == 3 and g[2].q1 < 0
    assert max_dev(sv_of(3, g), sv_of(3, F.fuse_qasm(text.replace("h q[0];", ""))[1][:2]
                                      + [F.FusedGate(0, -1, np.array([[1, 1], [1, -1]]) / np.sqrt(2))])) <= 1e-12


def test_fusion_flipped_cx_orientation():
    n, g = F.fuse_qasm("OPENQASM 2.0; qreg q[2]; cx q[1],q[0];")
    assert len(g) == 1 and (g[0].q0, g[0].q1) == (0, 1) and g[0].flipped
    psi = np.zeros(4, dtype=complex)
    psi[1] = 1  # |01>: q1 = 1 controls q0
    out = dense_apply_2q(psi, g[0].matrix, 0, 1, 2)
    assert abs(out[3] - 1) <= 1e-14


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_fusion_matches_oracle_on_random_circuits(oracle, seed):
    """fuse_circuit parity with the oracle restatement (fusion.cpp:79-135):
    identical block structure, matrices to rounding; and the fused list
    reproduces the raw circuit's statevector (test_circuit.cpp:169-177)."""
    n = 6
    oc = oracle.Circuit.random(n, 60, 1000 + seed, nonlocal_=True)
    og = oc.fuse().gates()
    n_, g = F.fuse_qasm(qasm_of(oc.ops(), n))
    assert n_ == n and len(g) == len(og)
    for a, (q0, q1, fl, m) in zip(g, og):
        assert (a.q0, a.q1, a.flipped) == (q0, q1, fl)
        assert np.abs(a.matrix - m).max() <= 1e-14
        assert np.abs(a.matrix.conj().T @ a.matrix - np.eye(len(m))).max() <= 1e-10
    assert max_dev(sv_of(n, g), oc.statevector()) <= 1e-12


@pytest.mark.parametrize("haar", [False, True])
def test_brickwork_generator_matches_oracle(oracle, haar):
    """brickwork_qasm (generators.cpp:95-145): the same angles to the bit
    (%.17g) and, for Haar entanglers, the same seeded 4x4 unitaries (sidecar,
    injected at their op positions) as the oracle's generator."""
    n, depth, seed = 7, 4, 4242
    qasm, sc = F.brickwork_qasm(n, depth, seed, entangler="haar" if haar else "cx")
    oc = oracle.Circuit.brickwork(n, depth, seed, haar=haar)
    c = F.parse_qasm(qasm)
    ours = [(o.kind, o.q0, o.q1, tuple(o.params)) for o in c.ops]
    theirs = [op for op in oc.ops() if op[0] != "u4"]
    assert ours == theirs
    assert (sc is not None) == haar
    if haar:
        doc = json.loads(sc)
        assert doc["format"] == "u4-sidecar-v1"
        assert len(doc["entanglers"]) == sum(op[0] == "u4" for op in oc.ops())
    _, g = F.fuse_qasm(qasm, sc)
    og = oc.fuse().gates()
    assert len(g) == len(og)
    for a, (q0, q1, fl, m) in zip(g, og):
        assert (a.q0, a.q1) == (q0, q1)
        assert np.abs(a.matrix - m).max() <= 1e-13


def test_ghz_generator_text():
    assert F.ghz_qasm(3) == HDR + "qreg q[3];\nh q[0];\ncx q[0],q[1];\ncx q[1],q[2];\n"
    assert F.ghz_qasm(2, measure=True).endswith("creg c[2];\nh q[0];\ncx q[0],q[1];\nmeasure q -> c;\n")
    with pytest.raises(F.ConfigError):
        F.ghz_qasm(1)
    with pytest.raises(F.ConfigError):
        F.brickwork_qasm(4, 0)
    a, _ = F.brickwork_qasm(6, 3, 123)
    assert a == F.brickwork_qasm(6, 3, 123)[0] and a != F.brickwork_qasm(6, 3, 124)[0]


def test_sidecar_injection_positions():
    """test_runner.cpp:101-119: entanglers land at their op_index slots."""
    qasm, sc = F.brickwork_qasm(4, 2, 9, entangler="haar")
    plain = F.parse_qasm(qasm)
    doc = json.loads(sc)
    n, g = F.fuse_qasm(qasm, sc)
    assert len(plain.ops) == 8  # u3 on every qubit, twice
    assert len(doc["entanglers"]) == 3
    assert all(x.q1 < 0 or x.q1 == x.q0 + 1 for x in g)


@pytest.mark.parametrize("mutate,fragment", [
    (lambda d: d.update(format="v0"), "u4-sidecar-v1"),
    (lambda d: d["entanglers"][0]["matrix"][0].__setitem__(0, 2.0), "not unitary"),
    (lambda d: d["entanglers"][0].__setitem__("op_index", 10 ** 6), "beyond end"),
    (lambda d: d["entanglers"][0].__setitem__("qubits", [1, 1]), "out of range"),
    (lambda d: d["entanglers"][0]["matrix"].pop(), "16 entries"),
])
def test_sidecar_errors(mutate, fragment):
    qasm, sc = F.brickwork_qasm(4, 1, 3, entangler="haar")
    doc = json.loads(sc)
    mutate(doc)
    with pytest.raises(F.ConfigError, match=fragment):
        F.fuse_qasm(qasm, json.dumps(doc))
    with pytest.raises(F.ConfigError, match="malformed"):
        F.fuse_qasm(qasm, sc[:-5])


# --------------------------------------------------------- lowering/layers
# tests/test_circuit.cpp:201-296

def test_decompose_swap_chain_shape():
    layers = F.plan_layers([(0, 2, np.eye(4))], 3)
    flat = [g for L in layers for g in L]
    assert [(g.q0, g.q1) for g in flat] == [(0, 1), (1, 2), (0, 1)]


def test_layerize_disjoint_and_shared():
    one = F.plan_layers([(0, 1, np.eye(4)), (2, 3, np.eye(4)), (4, -1, np.eye(2))], 5)
    assert len(one) == 1 and len(one[0]) == 3
    assert len(F.plan_layers([(0, 1, np.eye(4)), (1, 2, np.eye(4))], 3)) == 2


@pytest.mark.parametrize("seed", [11, 12])
def test_plan_matches_oracle(oracle, seed):
    """decompose_nonlocal + layerize parity with the oracle: same lowered
    gates in the same layers, and no layer reuses a qubit."""
    n = 8
    oc = oracle.Circuit.random(n, 80, seed, nonlocal_=True)
    og = oc.fuse()
    low = og.decompose_nonlocal(n)
    lo, nl = low.layer_of()
    _, g = F.fuse_qasm(qasm_of(oc.ops(), n))
    layers = F.plan_layers(g, n)
    want = {}
    for (q0, q1, _f, m), L in zip(low.gates(), lo):
        want.setdefault(int(L), []).append((q0, q1, m))
    assert len(layers) == len(want) == nl
    for L, gl in enumerate(layers):
        used = set()
        for x in gl:
            for q in (x.q0, x.q1) if x.q1 >= 0 else (x.q0,):
                assert q not in used
                used.add(q)
        assert [(x.q0, x.q1) for x in gl] == [(a, b) for a, b, _ in want[L]]
        for x, (_, _, m) in zip(gl, want[L]):
            assert np.abs(x.matrix - m).max() <= 1e-14


# ----------------------------------------------------------- run_circuit
# validation happens before any device work (test_runner.cpp:121-147)

def test_run_config_validation():
    ghz = F.ghz_qasm(4)
    with pytest.raises(F.ConfigError, match="bond propagation"):
        F.run_circuit(ghz, backend="mps-parallel", nonlocal_method="bondprop")
    with pytest.raises(F.ConfigError, match="no circuit"):
        F.run_circuit()
    with pytest.raises(F.ConfigError, match="workers"):
        F.run_circuit(ghz, backend="mps-parallel", workers=0)
    with pytest.raises(F.ConfigError, match="cannot read"):
        F.run_circuit(qasm_path="/nonexistent/file.qasm")
    with pytest.raises(F.ConfigError, match="cutoff"):
        F.run_circuit(ghz, cutoff=1.0)
    with pytest.raises(F.ParseError):
        F.run_circuit("OPENQASM 2.0; qreg q[2]; frobnicate q[0];")


def test_exit_codes():
    assert F.exit_code_for_error(F.ConfigError("x")) == 1
    assert F.exit_code_for_error(F.ParseError("x", 1, 2)) == 2
    assert F.exit_code_for_error(F.NumericError("x")) == 3
    assert F.exit_code_for_error(RuntimeError("x")) == 1


def test_cli_generators_and_exit_codes(tmp_path):
    """tools/main.cpp subcommands: gen-ghz / gen-brickwork output, error exit codes."""
    import subprocess
    import sys
    root = __import__("os").path.dirname(__import__("os").path.dirname(__file__))

    def cli(*args):
        return subprocess.run([sys.executable, "-m", "paper_2601_04422_b200", *args], cwd=root,
                              capture_output=True, text=True, timeout=120)

    r = cli("gen-ghz", "--n", "3")
    assert r.returncode == 0 and r.stdout == F.ghz_qasm(3)
    out = tmp_path / "bw.qasm"
    r = cli("gen-brickwork", "--n", "5", "--depth", "2", "--seed", "7", "--entangler", "haar", "--out", str(out))
    assert r.returncode == 0
    q, sc = F.brickwork_qasm(5, 2, 7, entangler="haar")
    assert out.read_text() == q
    assert json.loads((tmp_path / "bw.qasm.u4.json").read_text()) == json.loads(sc)
    assert cli("gen-brickwork", "--n", "5", "--depth", "2", "--entangler", "haar").returncode == 1
    assert cli("run", "--qasm", str(tmp_path / "missing.qasm")).returncode == 1
    bad = tmp_path / "bad.qasm"
    bad.write_text("OPENQASM 2.0; qreg q[2]; foo q[0];")
    r = cli("run", "--qasm", str(bad))
    assert r.returncode == 2 and "line 1, column" in r.stderr
