"""pytest configuration: the `gpu` marker and shared fixtures.

`-m "not gpu"` runs here (no GPU): oracle pins against the reference's known
answers, host logic, C-ABI symbol checks and gloo multi-process tests.
`-m gpu` runs on a B200 through the C-ABI (libcpdgpu.so)."""
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libcpdgpu.so)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    import oracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_1204_1586_b200 import build as B
    B.build()
    import paper_1204_1586_b200 as cpd
    ctx = cpd.Context(int(os.environ.get("CPDGPU_DEVICE", "0")))
    yield ctx
    ctx.close()
