"""Generates the committed golden fixtures tests/golden/grad_*.npz.

Inputs: the reference fixtures' Uniform01 stream (rng.hpp:16-26, reproduced
bit-for-bit by oracle/cpd_oracle.c) and the shared counter-based N(0,1)
generator.  Outputs: the all-mode gradients from the CPU oracle (a restatement
of mttkrp.cpp:113-253) cross-checked here against the entrywise definition
(test_util.hpp:44-60) before they are written.  Run from the repo root:
    python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1] / "oracle"))
import oracle as O  # noqa: E402

CASES = [
    # name, dims, R, generator
    ("t8_ones", [2, 2, 2], 2, "t8"),
    ("u01_2x3x4_r3", [2, 3, 4], 3, "u01"),
    ("u01_4x3x2_r3", [4, 3, 2], 3, "u01"),
    ("u01_2x3x2x4_r1", [2, 3, 2, 4], 1, "u01"),
    ("u01_5x3x4_r2", [5, 3, 4], 2, "u01"),
    ("nrm_6x7x8x9_r5", [6, 7, 8, 9], 5, "normal"),
    ("nrm_3x4x5x2x3_r4", [3, 4, 5, 2, 3], 4, "normal"),
    ("nrm_11x13_r7", [11, 13], 7, "normal"),
]


def main():
    for name, dims, R, gen in CASES:
        n = int(np.prod(dims))
        if gen == "t8":
            y = np.arange(1, 9, dtype=float)
            f = [np.ones((2, 2)) for _ in dims]
        elif gen == "u01":
            y = O.random_tensor(dims, 100 + R)
            f = O.random_factors(dims, R, 200 + R)
        else:
            y = O.fill_normal(7, n)
            f = [O.fill_normal(8 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(dims)]
        g, _, _ = O.cp_gradient_all(y, dims, f)
        for k in range(len(dims)):
            b = O.brute_mttkrp(y, dims, f, k + 1)
            assert np.abs(g[k] - b).max() <= 1e-12 * max(np.abs(b).max(), 1e-30), (name, k)
        out = {"dims": np.array(dims), "y": y}
        for k in range(len(dims)):
            out[f"A{k}"] = np.asfortranarray(f[k])
            out[f"G{k}"] = np.asfortranarray(g[k])
        np.savez_compressed(HERE / f"grad_{name}.npz", **out)
        print("wrote", name)


if __name__ == "__main__":
    main()
