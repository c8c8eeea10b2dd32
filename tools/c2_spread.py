"""C2 (64-qubit Haar brickwork, depth 20, chi 128, cutoff 1e-12): amplitude
spread between three CPU SVDs (LAPACK zgesdd / zgesvj / zgesvd) and the GPU,
on the 64 seeded bitstrings of tests/test_gpu_fullsize.py::test_c2_full_size.
Test-infrastructure diagnostic (imports the oracle)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # noqa: E402
import paper_2601_04422_b200 as gpu  # noqa: E402


def main():
    n, chi = 64, 128
    workers = os.cpu_count() or 1
    haar = "cx" not in sys.argv[1:]
    fused = oracle.Circuit.brickwork(n, 20, 4242, haar=haar).fuse()
    rng = np.random.default_rng(7)
    bits = ["".join(rng.choice(["0", "1"], n)) for _ in range(64)]
    amps, ks = {}, {}
    for b in ("zgesdd", "zgesvj", "zgesvd"):
        oracle.set_svd_backend(b)
        o = oracle.MpsState(n)
        r = oracle.execute_parallel(o, fused, chi, 1e-12, workers=workers)
        amps[b] = np.array([o.amplitude(x) for x in bits])
        ks[b] = r["gate_k"]
    oracle.set_svd_backend("zgesdd")
    g = gpu.MpsState(n, chi_hint=chi)
    rg = gpu.execute(g, [(q0, q1, m) for (q0, q1, _f, m) in fused.gates()], chi, 1e-12)
    amps["gpu"] = g.amplitudes(bits)
    ks["gpu"] = rg["gate_k"]
    ao = amps["zgesdd"]
    big = np.abs(ao) > 1e-14 * np.abs(ao).max()
    for b in ("zgesvj", "zgesvd", "gpu"):
        e = np.abs(amps[b][big] - ao[big]) / np.abs(ao[big])
        print(f"{b:7s} vs zgesdd: k equal {bool((ks[b] == ks['zgesdd']).all())}, amp rel err max {e.max():.3e} median {np.median(e):.3e}")
    e = np.abs(amps["gpu"][big] - amps["zgesvj"][big]) / np.abs(amps["zgesvj"][big])
    print(f"gpu     vs zgesvj: max {e.max():.3e}")


if __name__ == "__main__":
    main()
