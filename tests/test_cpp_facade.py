"""The header-only C++ facade (include/mpsim_b200.hpp) compiles against the C
ABI here and runs its host-only front-end checks (parse / fuse / plan /
generate), and runs its reference-style known answers on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "facade_test.cpp")
LIBDIR = os.path.join(ROOT, "paper_2601_04422_b200")
OUT = os.path.join(ROOT, "tests", "cpp", "facade_test")


def _compile():
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                    SRC, "-o", OUT, "-L", LIBDIR, "-lmpsim_gpu", f"-Wl,-rpath,{LIBDIR}"], check=True)


def test_facade_compiles():
    if not os.path.exists(os.path.join(LIBDIR, "libmpsim_gpu.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(LIBDIR, "csrc"), "-j8"], check=True)
    _compile()
    assert os.path.exists(OUT)
    out = subprocess.run([OUT, "--host-only"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "facade host ok" in out.stdout


@pytest.mark.gpu
def test_facade_runs_on_gpu():
    _compile()
    out = subprocess.run([OUT], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "facade ok" in out.stdout


@pytest.mark.gpu
def test_cpp_sharded_chain_world1(tmp_path):
    """The C++ facade's ShardedChain (csrc/shard.cu through mpsim_b200.hpp) at
    world size 1 against MpsState: bit-identical amplitudes, norm and sample
    counts (tools/r2_gpu3.sh / profiles run the same program at N = 2)."""
    src = os.path.join(ROOT, "tests", "cpp", "shard_main.cpp")
    exe = os.path.join(ROOT, "tests", "cpp", "shard_main")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                    src, "-o", exe, "-L", LIBDIR, "-lmpsim_gpu", f"-Wl,-rpath,{LIBDIR}"], check=True)
    out = subprocess.run([exe, "0", "1", str(tmp_path / "id"), "0"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "shard ok" in out.stdout
