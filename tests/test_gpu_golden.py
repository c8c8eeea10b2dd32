"""GPU path against the committed oracle fixtures of the BASELINE configs that
do not fit a live oracle run inside a test (tests/golden/make_golden.py):

  c3_full.npz    C3 at its stated size: 100-qubit brickwork depth 32 with
                 SWAP-routed non-adjacent CX gates, chi = 512, cutoff 1e-12
  c4_window.npz  a C4 window: 24-qubit disordered TFIM Trotter steps until the
                 centre bond reaches chi = 1024, then two more

The local gate list (SWAPs included) goes through the public execute path;
per-gate kept ranks must equal the oracle's exactly (SWAPs included);
discarded weights, amplitudes and <Z_q> / <X_q> agree to 1e-10 (relative,
relative, absolute) or to twice the oracle's own whole-circuit spread between
zgesdd and a second SVD when the header records a larger one (C3: after 1302
truncating gates two correct SVDs leave amplitudes 4.4x apart). The fixture's own header records that the oracle's zgesdd run and an
independent zgesvj (one-sided Jacobi) run agree on every kept rank."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
PZ = np.diag([1.0, -1.0]).astype(np.complex128)
PX = np.array([[0, 1], [1, 0]], dtype=np.complex128)


def _load(name):
    f = np.load(os.path.join(HERE, name + ".npz"))
    with open(os.path.join(HERE, name + ".json")) as fh:
        meta = json.load(fh)
    gates = []
    for q0, q1, m in zip(f["q0"], f["q1"], f["mats"]):
        gates.append((int(q0), int(q1), m if q1 >= 0 else m[:2, :2]))
    return f, meta, gates


def test_fixture_headers_pin_the_oracle():
    """CPU-side sanity (runs with -m gpu only because the fixture is GPU
    parity data): the zgesdd oracle and the independent zgesvj run agree."""
    for name in ("c3_full", "c4_window"):
        with open(os.path.join(HERE, name + ".json")) as fh:
            meta = json.load(fh)
        chk = meta["zgesvj_check"]
        assert chk["kept_ranks_equal"] and chk["bonds_equal"], name
        assert chk["max_rel_w_diff"] <= 1e-8, name  # (whole-circuit drift; see tests/test_golden_fixtures.py)
        if "svd_pin_summary" in meta:  # per-theta pins: the SVD decisions themselves
            assert meta["svd_pin_summary"]["max_w_rel_diff_w_above_1e-10"] <= 1e-10, name


def _run(gpu, name, known_deviation=None):
    """known_deviation: reason string; then kept ranks, bonds and <Z>/<X> are
    asserted strictly and a weight / amplitude excess over the tolerance is
    reported as an expected failure naming the measured values."""
    f, meta, gates = _load(name)
    # 1e-10 relative, or twice the spread between the oracle's two independent
    # SVDs (zgesdd vs zgesvj) where the truncated chain's conditioning already
    # separates them by more (see tests/test_gpu_fullsize.py C2)
    amp_tol = max(1e-10, 2.0 * meta["zgesvj_check"]["max_rel_amp_diff"])
    w_tol = max(1e-10, 2.0 * meta["zgesvj_check"]["max_rel_w_diff"])
    n, chi, cutoff = int(f["n"]), int(f["chi"]), float(f["cutoff"])
    g = gpu.MpsState(n, chi_hint=chi)
    rg = gpu.execute(g, gates, chi, cutoff)
    k, w = f["k"], f["w"]
    mism = np.nonzero(rg["gate_k"] != k)[0]
    assert mism.size == 0, (name, mism[:10], rg["gate_k"][mism[:10]], k[mism[:10]])
    assert rg["peak_bond"] == chi == k.max()
    nz = w > 1e-16  # below: rank-deficient rounding noise
    assert (rg["gate_w"][~nz] <= 1e-16).all()
    assert (g.bond_dims() == f["bonds"]).all()
    chk = meta["zgesvj_check"]
    zx_tol = {id(PZ): max(1e-10, 2.0 * chk.get("max_abs_z_diff", 0.0)),
              id(PX): max(1e-10, 2.0 * chk.get("max_abs_x_diff", 0.0))}
    for q, z, x in zip(f["qs"], f["z"], f["x"]):
        for op, ref in ((PZ, z), (PX, x)):
            got = g.expect_1q(op, int(q))
            assert abs(got - ref) <= zx_tol[id(op)] * max(1.0, abs(ref)), (name, int(q), got, ref, zx_tol[id(op)])
    w_err = float(np.max(np.abs(rg["gate_w"][nz] - w[nz]) / w[nz])) if nz.any() else 0.0
    ag = g.amplitudes([str(b) for b in f["bits"]])
    ao = f["amps"]
    a_err = float(np.max(np.abs(ag - ao) / np.abs(ao)))
    if known_deviation is not None and (w_err > w_tol or a_err > amp_tol):
        pytest.xfail(f"{known_deviation}: max rel w error {w_err:.2e}, max rel amplitude error {a_err:.2e} "
                     f"(tolerances {w_tol:.1e} / {amp_tol:.1e}); ranks, bonds, <Z>, <X> within tolerance")
    assert w_err <= w_tol, (name, w_err, w_tol)
    assert a_err <= amp_tol, (name, a_err, amp_tol)
    return rg


@pytest.mark.slow
def test_c3_full_size_against_fixture(gpu):
    rg = _run(gpu, "c3_full")
    assert rg["svd_count"].sum() == len(rg["gate_k"])  # every local gate (SWAPs too) is one SVD (P6)


@pytest.mark.slow
def test_c4_window_reaching_chi1024_against_fixture(gpu):
    # (weights 7e-14, <Z>/<X> 1.5e-14, amplitudes 7e-11 measured; before the
    # quadratic-phase exit was tightened to 1e-12 and the kept-vector
    # orthonormalisation was added: 2.2e-10 / 1.5e-11 / 2.9e-8)
    _run(gpu, "c4_window")
