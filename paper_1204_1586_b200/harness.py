"""The reference's benchmark harness and gradcheck flow on the device (SURVEY
§8(f) row 4): bench.hpp / bench.cpp (run_benchmark, the stable CSV columns) and
cpd_main.cpp:63-120 (gradcheck), with the ALS engines running on the B200.

    python -m paper_1204_1586_b200.harness bench --dims 10,10,10 --rank 10 --iters 20 --csv out.csv
    python -m paper_1204_1586_b200.harness gradcheck --dims 4,5,6 --rank 3 --trials 3

Times are device-timed sweeps (the trace's CUDA-event seconds), as the
reference times sweeps only (als.cpp:176-192)."""
from __future__ import annotations

import argparse
import math
import sys
from dataclasses import dataclass, field
from typing import Optional, Sequence, TextIO

import numpy as np

from . import api, errors

CSV_HEADER = "N,dims,R,iters,reps,t_direct,t_fast,rho,mults_direct,mults_fast,count_ratio"


@dataclass
class BenchConfig:
    """bench.hpp:14-24."""
    dims: list = field(default_factory=list)  # empty selects the built-in grid
    rank: int = 10
    iters: int = 20
    reps: int = 0  # 0 picks max(1, ceil(200 / iters))
    seed: int = 42
    baseline: str = "als_direct"
    accelerated: str = "als_fast"
    match_order: bool = False  # run the baseline in the pivot update order
    mem_budget: int = 1 << 30


@dataclass
class BenchRecord:
    """bench.hpp:29-42."""
    dims: list
    rank: int
    iters: int
    reps: int
    t_baseline: float = 0.0
    t_fast: float = 0.0
    rho: float = 0.0
    rho_mean_of_ratios: float = 0.0
    per_rep_rho: list = field(default_factory=list)
    mults_baseline: int = 0
    mults_fast: int = 0
    count_ratio: float = 0.0


def speed_ratio(t_als: float, t_fast: float) -> float:
    """bench.cpp:139-143."""
    if not (t_als > 0.0) or not (t_fast > 0.0):
        raise errors.ArgumentError("speed_ratio: times must be positive")
    return t_als / t_fast


def _prefix(dims):
    J = [1]
    for d in dims:
        J.append(J[-1] * int(d))
    return J


def _sum_j_prefix(J, lo, hi, div=1):
    return sum(J[k] // div for k in range(lo, hi + 1)) if lo <= hi else 0


def predicted_mult_count(dims: Sequence[int], R: int, n: int, variant: str) -> int:
    """predicted_mult_count (mttkrp.cpp:255-290) on ascending dims; variant is
    direct, fast or fast_derived."""
    dims = [int(d) for d in dims]
    N = len(dims)
    if not 1 <= n <= N:
        raise errors.IndexError(f"predicted_mult_count: mode {n} outside 1..{N}")
    if R < 1:
        raise errors.ArgumentError("predicted_mult_count: rank must be positive")
    if dims != sorted(dims):
        raise errors.ArgumentError("predicted_mult_count: dims must be ascending")
    J = _prefix(dims)
    if variant == "direct":
        return R * (J[N] + _sum_j_prefix(J, 2, n - 1) + _sum_j_prefix(J, n + 1, N, dims[n - 1]))
    p = api.select_pivot(dims)
    if n in (p, p + 1):
        pivot_term = min(J[n], J[N] // J[n - 1])
        return R * (_sum_j_prefix(J, 2, n - 1) + pivot_term + _sum_j_prefix(J, n + 2, N, J[n]) + J[N])
    if n < p:
        return R * _sum_j_prefix(J, 2, n + 1)
    tail = _sum_j_prefix(J, n + 2, N) if variant == "fast" else _sum_j_prefix(J, n + 2, N, J[n])
    return R * (J[N] // J[n - 2] + J[N] // J[n - 1] + tail)


def predicted_sweep_counts(dims: Sequence[int], rank: int) -> tuple:
    """bench.cpp:25-35: analytic per-sweep totals on the ascending frame."""
    sd = sorted(int(d) for d in dims)
    direct = sum(predicted_mult_count(sd, rank, n, "direct") for n in range(1, len(sd) + 1))
    fast = sum(predicted_mult_count(sd, rank, n, "fast") for n in range(1, len(sd) + 1))
    return direct, fast


def estimate_cell_bytes(dims: Sequence[int], rank: int) -> int:
    """bench.cpp:145-160: working-set estimate used by the memory budget cap."""
    sd = sorted(int(d) for d in dims)
    J = _prefix(sd)
    jn, r = J[-1], int(rank)
    p = api.select_pivot(sd) if len(sd) >= 2 else 1
    fast_ws = r * (J[p] + jn // J[p]) if len(sd) >= 2 else r
    direct_ws = r * (jn // sd[0])
    factor_doubles = sum(d * r for d in sd)
    return 8 * (2 * jn + max(fast_ws, direct_ws) + 4 * factor_doubles)


def default_grid() -> list:
    """bench.cpp:104-112: N = 3..7, I in {10, 20}, R = 1, 10, 20, ... <= I."""
    cells = []
    for n in range(3, 8):
        for i in (10, 20):
            r = 1
            while r <= i:
                cells.append(([i] * n, r))
                r = 10 if r == 1 else r + 10
    return cells


def _run_rep(y, init, algo, cfg, ctx):
    opts = api.SolveOptions(max_iters=cfg.iters, tol=0.0)
    if cfg.match_order and algo == cfg.baseline:
        opts.order = "pivot"
    counter = api.CostCounter()
    res = api.run(y, init, opts, counter=counter, algo=algo)
    return float(sum(res.trace.seconds)), counter.total()


def run_cell(dims, rank, reps, cfg, ctx=None) -> BenchRecord:
    """bench.cpp:59-94."""
    rec = BenchRecord(dims=list(dims), rank=rank, iters=cfg.iters, reps=reps)
    tb = tf = 0.0
    mb = mf = 0
    for rep in range(reps):
        y, init = api.generate_problem(dims, rank, cfg.seed + 2 * rep, ctx=ctx)
        b = _run_rep(y, init, cfg.baseline, cfg, ctx)
        f = _run_rep(y, init, cfg.accelerated, cfg, ctx)
        y.free()
        tb += b[0]
        tf += f[0]
        mb += b[1]
        mf += f[1]
        rec.per_rep_rho.append(speed_ratio(b[0], f[0]))
    per_iter = reps * cfg.iters
    rec.t_baseline, rec.t_fast = tb / per_iter, tf / per_iter
    rec.rho = speed_ratio(rec.t_baseline, rec.t_fast)
    rec.rho_mean_of_ratios = float(np.mean(rec.per_rep_rho))
    rec.mults_baseline, rec.mults_fast = mb // per_iter, mf // per_iter
    pd, pf = predicted_sweep_counts(dims, rank)
    rec.count_ratio = pd / pf
    return rec


def run_benchmark(cfg: BenchConfig, log: Optional[TextIO] = None, ctx=None) -> list:
    """bench.cpp:162-182: every cell of the grid (or cfg.dims), skipping cells over
    the memory budget and reporting per-cell failures on `log`."""
    if cfg.iters < 1:
        raise errors.ArgumentError("run_benchmark: iters must be at least 1")
    if cfg.reps < 0:
        raise errors.ArgumentError("run_benchmark: reps must be nonnegative")
    if any(int(d) < 1 for d in cfg.dims):
        raise errors.ArgumentError("run_benchmark: dims must be at least 1")
    reps = cfg.reps if cfg.reps > 0 else max(1, math.ceil(200 / cfg.iters))
    cells = default_grid() if not cfg.dims else [(list(cfg.dims), cfg.rank)]
    records = []
    for dims, rank in cells:
        label = "x".join(map(str, dims))
        need = estimate_cell_bytes(dims, rank)
        if need > cfg.mem_budget:
            if log:
                log.write(f"skip {label} R={rank}: needs ~{need} bytes, budget {cfg.mem_budget}\n")
            continue
        try:
            records.append(run_cell(dims, rank, reps, cfg, ctx))
        except Exception as e:  # noqa: BLE001 - reported and skipped, as the reference does
            if log:
                log.write(f"cell {label} R={rank} failed: {e}\n")
    return records


def write_csv(out: TextIO, records: Sequence[BenchRecord]) -> None:
    """bench.cpp:184-196: the stable column set."""
    out.write(CSV_HEADER + "\n")
    for r in records:
        out.write(f"{len(r.dims)},{'x'.join(map(str, r.dims))},{r.rank},{r.iters},{r.reps},"
                  f"{r.t_baseline:.9g},{r.t_fast:.9g},{r.rho:.6g},{r.mults_baseline},{r.mults_fast},"
                  f"{r.count_ratio:.6g}\n")


def write_table(out: TextIO, records: Sequence[BenchRecord]) -> None:
    out.write(f"{'dims':<16s} {'R':>4s} {'iters':>6s} {'reps':>4s} {'t_direct':>12s} {'t_fast':>12s} "
              f"{'rho':>8s} {'cnt':>8s}\n")
    for r in records:
        out.write(f"{'x'.join(map(str, r.dims)):<16s} {r.rank:>4d} {r.iters:>6d} {r.reps:>4d} "
                  f"{r.t_baseline:>12.4e} {r.t_fast:>12.4e} {r.rho:>8.3f} {r.count_ratio:>8.3f}\n")


def gradcheck(dims: Sequence[int], rank: int, trials: int = 3, seed: int = 42, out: TextIO = sys.stdout,
              ctx=None) -> int:
    """cpd_main.cpp:63-120: per trial, fast vs direct MTTKRP (<= 1e-12 of the largest
    entry) and central differences of the cost against the stacked gradient (<= 1e-5)."""
    failures = 0
    for t in range(trials):
        y, init = api.generate_problem(dims, rank, seed + 2 * t, ctx=ctx)
        fast = api.cp_gradient_all(y, init)
        worst = 0.0
        for n in range(1, len(dims) + 1):
            direct = api.mttkrp_direct(y, init, n)
            scale = max(np.abs(direct).max(), 1e-30)
            worst = max(worst, np.abs(direct - fast[n - 1]).max() / scale)
        equiv_ok = worst <= 1e-12
        modes, g = api.cp_gradient_set(y, init, fast)
        gmax = np.abs(g).max()
        probe = [a.copy(order="F") for a in init]
        fd_worst = 0.0
        flat = 0
        for mode in range(len(probe)):
            A = probe[mode]
            for c in range(A.shape[1]):
                for i in range(A.shape[0]):
                    save = A[i, c]
                    h = 1e-6 * max(1.0, abs(save))
                    A[i, c] = save + h
                    dp = api.cost(y, probe)
                    A[i, c] = save - h
                    dm = api.cost(y, probe)
                    A[i, c] = save
                    fd = (dp - dm) / (2.0 * h)
                    an = g[flat]
                    fd_worst = max(fd_worst, abs(fd - an) / max(abs(fd), abs(an), 1e-8 * gmax))
                    flat += 1
        fd_ok = fd_worst <= 1e-5
        out.write(f"trial {t + 1:2d}: fast-vs-direct {worst:.3e} {'ok' if equiv_ok else 'FAIL'}, "
                  f"finite-diff {fd_worst:.3e} {'ok' if fd_ok else 'FAIL'}\n")
        if not (equiv_ok and fd_ok):
            failures += 1
        y.free()
    if failures:
        out.write(f"{failures} of {trials} trials failed\n")
        return 1
    out.write(f"all {trials} trials passed\n")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1204_1586_b200.harness")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench")
    b.add_argument("--dims", default="")
    b.add_argument("--rank", type=int, default=10)
    b.add_argument("--iters", type=int, default=20)
    b.add_argument("--reps", type=int, default=0)
    b.add_argument("--seed", type=int, default=42)
    b.add_argument("--match-order", action="store_true")
    b.add_argument("--csv", default="")
    g = sub.add_parser("gradcheck")
    g.add_argument("--dims", required=True)
    g.add_argument("--rank", type=int, default=3)
    g.add_argument("--trials", type=int, default=3)
    g.add_argument("--seed", type=int, default=42)
    a = ap.parse_args(argv)
    dims = [int(x) for x in a.dims.split(",") if x]
    if a.cmd == "gradcheck":
        return gradcheck(dims, a.rank, a.trials, a.seed)
    cfg = BenchConfig(dims=dims, rank=a.rank, iters=a.iters, reps=a.reps, seed=a.seed, match_order=a.match_order)
    recs = run_benchmark(cfg, log=sys.stderr)
    write_table(sys.stdout, recs)
    if a.csv:
        with open(a.csv, "w") as f:
            write_csv(f, recs)
    return 0


if __name__ == "__main__":
    sys.exit(main())
