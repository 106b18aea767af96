"""Small gradients through every seed pipeline, for compute-sanitizer runs
(tests/test_gpu_sanitizer.py): the int8 fused pass (forced), the fp64 DMMA
pass, the fused fp32 pass on the operand image, the fused fp32 pass splitting
in-kernel, the two-pass fp32 path (a hook), and one fast ALS sweep.  Each result
is checked against the CPU oracle so a run that "passes" the sanitizer also
computed the right numbers.  Usage: python tests/sanitize_cases.py [case...]"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def main(cases):
    import oracle as O
    import paper_1204_1586_b200 as cpd
    ctx = cpd.Context(0)
    assert ctx._L.cpdgpu_set_graphs(ctx.h, 0) == 0  # eager launches: every kernel is seen as launched

    def check(g, want, tol):
        for a, b in zip(g, want):
            err = np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
            assert err <= tol, err

    for case in cases:
        if case in ("i8", "f64"):
            os.environ["CPDGPU_I8"] = "1" if case == "i8" else "0"
            dims, R = [16, 12, 10, 8], 5
            y = cpd.DenseTensor.generate(dims, cpd.DIST_NORMAL, seed=3, ctx=ctx)
            f = [O.fill_normal(40 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(dims)]
            g = cpd.cp_gradient_all(y, f)
            assert ctx.last_seed_path() == (1 if case == "i8" else 0)
            check(g, O.cp_gradient_all(y.values(), dims, f)[0], 1e-10)
            del os.environ["CPDGPU_I8"]
        elif case in ("f32i", "f32f", "f32hook"):
            if case == "f32f":
                os.environ["CPDGPU_F32_IMAGE"] = "0"
            dims, R = [20, 20, 20, 20], 64
            y = cpd.DenseTensor.generate(dims, cpd.DIST_UNIFORM_PM1, seed=3, ctx=ctx, dtype=cpd.F32)
            f = [O.fill_normal(50 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(dims)]
            if case == "f32hook":
                g = cpd.cp_gradient_all(y, f, hook=lambda n, G: None)
            else:
                g = cpd.cp_gradient_all(y, f)
                assert ctx.last_seed_path() == (4 if case == "f32i" else 3), ctx.last_seed_path()
            check(g, O.cp_gradient_all(y.values().astype(np.float64), dims, f)[0], 1e-5)
            os.environ.pop("CPDGPU_F32_IMAGE", None)
        elif case == "als":
            dims, R = [10, 11, 12], 4
            y = cpd.DenseTensor.generate(dims, cpd.DIST_NORMAL, seed=9, ctx=ctx)
            f = [O.fill_normal(60 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(dims)]
            f2 = [x.copy(order="F") for x in f]
            cpd.als_sweep_fast(y, f2)
            O.als_sweep_fast(y.values(), dims, f)
            for a, b in zip(f2, f):
                assert np.abs(a - b).max() <= 1e-9 * max(np.abs(b).max(), 1.0)
        else:
            raise SystemExit(f"unknown case {case}")
        print("ok", case, flush=True)
    ctx.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["i8", "f64", "f32i", "f32f", "f32hook", "als"])
