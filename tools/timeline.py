"""Launch timeline of the device gradient (CPDGPU_TIMELINE=1): per kernel the
earliest CTA entry, the earliest return from its dependency wait and the last
warp exit, in microseconds from the prologue's first CTA (graph replay)."""
import os, subprocess, sys
os.environ["CPDGPU_TIMELINE"] = "1"
# the stamps are compiled in only with -DCPDGPU_TIMELINE: use a variant library
_root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_lib = os.path.join(_root, "tools", "bisect_timeline.so")
if "CPDGPU_LIB" not in os.environ:
    if not os.path.exists(_lib):
        subprocess.run([sys.executable, os.path.join(_root, "tools", "build_variant.py"), "timeline", "-",
                        "-DCPDGPU_TIMELINE"], check=True)
    os.environ["CPDGPU_LIB"] = _lib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1204_1586_b200 as cpd
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
dims, R = {"c1": ([200] * 3, 10), "c2": ([60] * 4, 20), "c3": ([14] * 7, 10), "c5": ([300] * 4, 64)}[cfg]
ctx = cpd.Context(0)
y = (cpd.DenseTensor.generate(dims, cpd.DIST_UNIFORM_PM1, seed=1, ctx=ctx, dtype=cpd.F32) if cfg == "c5"
     else cpd.DenseTensor.generate(dims, cpd.DIST_NORMAL, seed=1, ctx=ctx))  # c5 is the fp32 config
f = [np.random.default_rng(k).normal(size=(d, R)) for k, d in enumerate(dims)]
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 6):
    cpd.cp_gradient_all(y, f)
