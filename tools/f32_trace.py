"""Per-warp wait/total cycle trace of the fp32 seed passes (CPDGPU_SEED_TRACE=1) on c5."""
import os, sys
os.environ["CPDGPU_SEED_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1204_1586_b200 as cpd
dims, R = [300] * 4, 64
ctx = cpd.Context(0)
y = cpd.DenseTensor.generate(dims, cpd.DIST_UNIFORM_PM1, seed=1, ctx=ctx, dtype=cpd.F32)
f = [np.random.default_rng(k).normal(size=(d, R)) for k, d in enumerate(dims)]
for _ in range(2):
    cpd.cp_gradient_all(y, f)
