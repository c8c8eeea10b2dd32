"""Adds the second-SVD spread of <Z_q>, <X_q> to the C3 fixture header
(TEST INFRASTRUCTURE): re-runs the fixture's gate list through the oracle with
LAPACK zgesvd (as make_golden.py's second run) and records
max |<O>_zgesvd - <O>_fixture| for O in {Z, X} as zgesvj_check.max_abs_z_diff /
max_abs_x_diff."""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import make_golden as M  # noqa: E402
from oracle import oracle as O  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3_full"
workers = int(sys.argv[2]) if len(sys.argv) > 2 else (os.cpu_count() or 1)
f = np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))
meta_path = os.path.join(ROOT, "tests", "golden", name + ".json")
meta = json.load(open(meta_path))
gates = [(int(a), int(b), m if b >= 0 else m[:2, :2]) for a, b, m in zip(f["q0"], f["q1"], f["mats"])]
gl = O.GateList(gates)
n, chi, cutoff = int(f["n"]), int(f["chi"]), float(f["cutoff"])
t0 = time.time()
O.set_svd_backend(meta["zgesvj_check"].get("second_svd", "zgesvd"))
o, k, w = M.run_oracle(n, gl, chi, cutoff, workers)
O.set_svd_backend("zgesdd")
_, _, z, x = M.observables(o, n, list(f["qs"]), workers)
meta["zgesvj_check"]["max_abs_z_diff"] = float(np.max(np.abs(z - f["z"])))
meta["zgesvj_check"]["max_abs_x_diff"] = float(np.max(np.abs(x - f["x"])))
meta["zgesvj_check"]["observable_spread_seconds"] = time.time() - t0
json.dump(meta, open(meta_path, "w"), indent=1)
print(name, "z spread", meta["zgesvj_check"]["max_abs_z_diff"], "x spread", meta["zgesvj_check"]["max_abs_x_diff"])
