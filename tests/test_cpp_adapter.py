"""The C++ drop-in adapter (include/cpd_gpu/cpd.hpp): the reference's cpd::
signatures over the C-ABI.  CPU: it compiles warning-free against the in-tree
library.  GPU: tests/cpp/test_adapter.cpp (reference-style KATs, fast == brute,
hook contract, counts, ALS) passes on the B200."""
import shutil
import subprocess
from pathlib import Path

import pytest

from paper_1204_1586_b200 import build as B

ROOT = Path(__file__).resolve().parents[1]
CPP = ROOT / "tests" / "cpp"


def _build(eigen=False):
    """eigen=True: CPD_GPU_WITH_EIGEN, cpd::Matrix = Eigen::MatrixXd, against the
    Eigen API subset shim (oracle/shim: this image has no Eigen) — the mode a
    reference user compiles the adapter in."""
    B.build()
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    out = CPP / "_build" / ("test_adapter_eigen" if eigen else "test_adapter")
    out.parent.mkdir(exist_ok=True)
    extra = ["-DCPD_GPU_WITH_EIGEN", f"-I{ROOT / 'oracle' / 'shim'}"] if eigen else []
    r = subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", *extra, f"-I{ROOT / 'include'}",
                        str(CPP / "test_adapter.cpp"), f"-L{B.LIB.parent}", "-lcpdgpu",
                        f"-Wl,-rpath,{B.LIB.parent}", "-o", str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


@pytest.mark.parametrize("eigen", [False, True])
def test_adapter_compiles(eigen):
    assert _build(eigen).exists()


@pytest.mark.gpu
@pytest.mark.parametrize("eigen", [False, True])
def test_adapter_suite_on_device(eigen):
    exe = _build(eigen)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
