"""In-tree build of the sm_100a shared library (no JIT cache, no pip install).

The library lands at paper_1204_1586_b200/lib/libcpdgpu.so so it travels to the
GPU box with the repository snapshot.  Compiled only for B200:
``-gencode arch=compute_100a,code=sm_100a``.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "lib"
LIB = LIB_DIR / "libcpdgpu.so"
INCLUDE = PKG.parent / "include"

SOURCES = ["cpdgpu.cu", "seed_f64.cu", "seed_i8.cu", "seed_f32.cu", "seed_f32f.cu", "tail.cu", "util.cu", "als.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def sources() -> list[Path]:
    return [CSRC / s for s in SOURCES if (CSRC / s).exists()]


def source_hash() -> str:
    import hashlib
    h = hashlib.sha256(" ".join(NVCC_FLAGS).encode())
    deps = sorted(sources() + list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh"))) + [INCLUDE / "cpdgpu.h"]
    for p in deps:
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()


HASH_FILE = LIB_DIR / "libcpdgpu.srchash"


def needs_build() -> bool:
    """Content hash, not mtimes: snapshots copied to the GPU box keep the prebuilt .so."""
    if not LIB.exists() or not HASH_FILE.exists():
        return True
    return HASH_FILE.read_text().strip() != source_hash()


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    LIB_DIR.mkdir(exist_ok=True)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, "-I", str(INCLUDE), "-o", str(tmp), *map(str, sources())]
    res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    log = res.stdout + res.stderr
    (LIB_DIR / "ptxas.log").write_text(log)
    if res.returncode != 0:
        sys.stderr.write(log)
        raise RuntimeError(f"nvcc failed ({res.returncode}); see {LIB_DIR / 'ptxas.log'}")
    os.replace(tmp, LIB)
    HASH_FILE.write_text(source_hash())
    if verbose:
        sys.stderr.write(log)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
