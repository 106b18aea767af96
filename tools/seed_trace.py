"""Per-warp cycle trace of the fp64 seed kernel (CPDGPU_SEED_TRACE=1) on a config."""
import os, sys
os.environ["CPDGPU_SEED_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1204_1586_b200 as cpd
dims, R = {"c1": ([200] * 3, 10), "c2": ([60] * 4, 20), "c3": ([14] * 7, 10)}[sys.argv[1]]
ctx = cpd.Context(0)
y = cpd.DenseTensor.generate(dims, cpd.DIST_NORMAL, seed=1, ctx=ctx)
f = [np.random.default_rng(k).normal(size=(d, R)) for k, d in enumerate(dims)]
for _ in range(3):
    cpd.cp_gradient_all(y, f)
