"""The committed oracle fixtures (tests/golden/, written by make_golden.py) on
CPU: the oracle re-run over a prefix of each fixture's gate list reproduces
the fixture's per-gate kept ranks and discarded weights, and each fixture's
header records that a second, independent SVD agreed on every kept rank.
The GPU side of the same fixtures is tests/test_gpu_golden.py."""
import json
import os

import numpy as np
import pytest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = [n for n in ("c3_full", "c4_window") if os.path.exists(os.path.join(HERE, n + ".npz"))]


def _load(name):
    f = np.load(os.path.join(HERE, name + ".npz"))
    with open(os.path.join(HERE, name + ".json")) as fh:
        meta = json.load(fh)
    gates = [(int(q0), int(q1), m if q1 >= 0 else m[:2, :2]) for q0, q1, m in zip(f["q0"], f["q1"], f["mats"])]
    return f, meta, gates


@pytest.mark.parametrize("name", NAMES)
def test_fixture_header(name):
    f, meta, gates = _load(name)
    assert len(gates) == len(f["k"]) == len(f["w"]) == meta["local_gates"]
    assert int(f["k"].max()) == meta["peak_bond"] == int(f["chi"])
    chk = meta["zgesvj_check"]
    assert chk["kept_ranks_equal"] and chk["bonds_equal"] and chk["rank_mismatches"] == 0
    # whole-circuit drift between the two SVDs: recorded, it sets the GPU test's
    # weight / amplitude tolerances (twice it, floor 1e-10). Measured: c4 5e-14 /
    # 7e-12; c3 (3120 gates, 1302 truncating at chi = 512) 1.1e-9 / 4.4 — after
    # that many truncations two correct SVDs leave different amplitudes (P10)
    assert np.isfinite(chk["max_rel_w_diff"]) and chk["max_rel_w_diff"] <= 1e-8
    if "svd_pin_summary" in meta:
        assert meta["svd_pin_summary"]["kept_ranks_equal"]
        assert meta["svd_pin_summary"]["max_w_rel_diff_w_above_1e-10"] <= 1e-10
    assert len(f["bits"]) == len(f["amps"]) == 64
    assert np.all(np.isfinite(f["amps"])) and np.all(np.abs(f["amps"]) > 0)


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_fixture_prefix(name, oracle):
    """Gate by gate (execute_serial; the per-gate inputs equal the layered
    run's) over the prefix whose bonds stay <= 64: kept ranks exactly, weights
    to 1e-12 (the same oracle, the same LAPACK)."""
    f, meta, gates = _load(name)
    n = int(f["n"])
    k = f["k"]
    stop = int(np.argmax(k > 64)) if (k > 64).any() else len(gates)
    stop = min(stop, 600)
    o = oracle.MpsState(n)
    r = oracle.execute_serial(o, oracle.GateList(gates[:stop]), int(f["chi"]), float(f["cutoff"]))
    assert (r["gate_k"] == k[:stop]).all()
    w = f["w"][:stop]
    nz = w > 1e-16
    if nz.any():
        assert np.max(np.abs(r["gate_w"][nz] - w[nz]) / w[nz]) <= 1e-12
