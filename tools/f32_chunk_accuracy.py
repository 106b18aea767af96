"""How long may an fp32 TMEM accumulator run before its drain?  Relative
Frobenius error of the fp32 tensor-core gradient against the fp64 streaming
oracle at config 5 (both seeds sum K = 90000 terms), as a
function of CPDGPU_F32_CHUNK (k-tiles of 64 columns per TMEM accumulation
window).  Usage: python tools/f32_chunk_accuracy.py [chunk ...]"""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
DIMS, R, SEED = [300, 300, 300, 300], 64, 7


def factors(O):
    return [O.fill_normal(500 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(DIMS)]


def child(out):
    import paper_1204_1586_b200 as cpd
    import oracle as O
    ctx = cpd.Context(0)
    y = cpd.DenseTensor.generate(DIMS, cpd.DIST_UNIFORM_PM1, seed=SEED, ctx=ctx, dtype=cpd.F32)
    g = cpd.cp_gradient_all(y, factors(O))
    np.savez(out, *g)


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--child":
        return child(sys.argv[2])
    import oracle as O
    want = O.cp_gradient_all_upm1_f32(DIMS, SEED, factors(O))
    for ch in (sys.argv[1:] or ["4", "8", "32", "128", "512", "1407"]):
        out = f"/tmp/f32acc_{ch}.npz"
        subprocess.run([sys.executable, __file__, "--child", out], check=True,
                       env={**os.environ, "CPDGPU_F32_CHUNK": ch})
        got = np.load(out)
        errs = [float(np.linalg.norm(got[f"arr_{k}"] - want[k]) / np.linalg.norm(want[k])) for k in range(4)]
        print(f"chunk {ch:>5} ({int(ch) * 64} columns): rel Frobenius per mode", " ".join(f"{e:.2e}" for e in errs),
              flush=True)


if __name__ == "__main__":
    main()
