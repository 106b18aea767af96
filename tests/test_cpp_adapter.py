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


def _build():
    B.build()
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    out = CPP / "_build" / "test_adapter"
    out.parent.mkdir(exist_ok=True)
    r = subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}",
                        str(CPP / "test_adapter.cpp"), f"-L{B.LIB.parent}", "-lcpdgpu",
                        f"-Wl,-rpath,{B.LIB.parent}", "-o", str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_adapter_compiles():
    assert _build().exists()


@pytest.mark.gpu
def test_adapter_suite_on_device():
    exe = _build()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
