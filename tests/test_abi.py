"""C-ABI surface checks that need no GPU: the library loads, exports every
symbol include/mpsim_gpu.h declares, and rejects bad arguments on the host
before touching a device."""
import ctypes
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ensure_built():
    lib = os.path.join(ROOT, "paper_2601_04422_b200", "libmpsim_gpu.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2601_04422_b200", "csrc"), "-j8"], check=True)
    return lib


def test_library_exports_every_declared_symbol():
    from paper_2601_04422_b200 import native
    path = _ensure_built()
    declared = native.exported_symbols()
    assert len(declared) >= 30
    handle = ctypes.CDLL(path)
    missing = [s for s in declared if not hasattr(handle, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    for s in declared:
        assert f" T {s}" in out, s


def test_binding_signatures_cover_header():
    from paper_2601_04422_b200 import native
    _ensure_built()
    L = native.lib()
    for s in native.exported_symbols():
        fn = getattr(L, s)
        assert fn.argtypes is not None or s == "mpsim_gpu_last_error", s


def test_kernels_target_sm100a():
    path = _ensure_built()
    out = subprocess.run(["cuobjdump", "-lelf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_null_state_is_rejected_without_a_device():
    from paper_2601_04422_b200 import native
    _ensure_built()
    L = native.lib()
    v = ctypes.c_int32()
    assert L.mpsim_gpu_num_qubits(None, ctypes.byref(v)) == native.MPSIM_EINVAL
    assert b"null" in L.mpsim_gpu_last_error()


def test_python_mirror_validates_shapes_on_host():
    from paper_2601_04422_b200 import mps
    with pytest.raises(ValueError):
        mps._cm([[1, 0], [0, 1]], 4)
    with pytest.raises(ValueError):
        mps.execute_parallel(None, [(0, 3, [[1] * 4] * 4)])
