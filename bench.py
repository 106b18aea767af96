#!/usr/bin/env python
"""Benchmark of the all-mode CP gradient on B200 (BASELINE.json metric).

A "step" is one all-mode CP gradient (cp_gradient_all) of the workload tensor.
Default workload (N=1): BASELINE.json configs[4] (c5), the largest config that
fits one GPU: the 300^4 fp32 tensor (32.4 GB, U(-1,1)) with R=64 N(0,1)
factors, synthetic inputs from the counter-based generator.  For N>1 (torchrun,
one rank per GPU) the same 300^4 tensor is sharded along its last mode (strong
scaling, 300 -> 38/38/38/38/37/37/37/37 at N=8): every rank's slab runs with the
global pivot, then one NCCL all_reduce of the partial G(1..3) carrying the G(4)
rows at each slab's offset, inside libcpdgpu.so (cpdgpu_comm_init from an NCCL id
broadcast over torch.distributed; paper_1204_1586_b200/sharded.py).  The fp64 configs
c1..c4 run with --config (c2, c3: weak scaling, one slab per GPU).

Timing: W untimed warm-up steps; then exactly K steps bracketed by a barrier +
cuda synchronize on both sides.  Tensors smaller than 4x the 256 MiB flush
buffer are preceded by an L2 flush (a 256 MiB device memset, outside the
events); c5's 32.4 GB tensor is far larger than L2.  Each step is timed with
CUDA events on the launching stream and the max over ranks of the summed step
time is reported.

  value      whole-job tensor bytes per second (GB/s) through the device API
  e2e        same metric through the host C-ABI (cpdgpu_cp_gradient_all): H2D
             copy of Y from pinned host memory + factors in, gradients out
  roofline   dominant kernel = K1 seed contraction, timed with CUDA events on the
             launching stream.  fp32 (c5): seed_f32i_kernel on tcgen05 kind::f16 over
             the fp16 hi/lo operand image, both seeds in one pass, bound = HBM.  Large fp64 tensors (c2, c3) run it on the int8 tensor cores
             (seed_i8_kernel): bound = HBM.  Otherwise fp64 DMMA
             (seed_f64_kernel, CPDGPU_I8=0 forces it): the slower of the HBM and
             FP64-tensor ideals, the other fraction beside it
             (e2e.pageable_upload: the upload rate from PAGEABLE host memory
             through the library's staged copy against a plain cudaMemcpy)
  cpu_baseline  the reference itself (oracle/_ref: its own sources built -O3
             -DNDEBUG over the Eigen shim), one single-threaded call per host
             core on mode-1 slabs of a bounded sample (kind "reference"); the C
             port of the reference (kind "port") only when that build is absent

`--impl reference` times the same reference build on all host cores on the same
workload and metric (the port as fallback).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (dims, R, dtype, description)
    "c1": ([200, 200, 200], 10, "f64", "3-D 200^3 fp64 R=10"),
    "c2": ([60, 60, 60, 60], 20, "f64", "4-D 60^4 fp64 R=20"),
    "c3": ([14] * 7, 10, "f64", "7-D 14^7 fp64 R=10"),
    # CP_ALS end to end: a step is one fast ALS sweep (BASELINE.json configs[3])
    "c4": ([60] * 5, 16, "f64", "5-D 60^5 fp64 rank-16 model + 20 dB noise, R=16"),
    # fp32 on the tensor cores; the 300^4 tensor is split over the GPUs (strong scaling)
    "c5": ([300] * 4, 64, "f32", "4-D 300^4 fp32 R=64"),
}
STRONG_CONFIGS = {"c5"}
ALS_CONFIGS = {"c4"}
C4_ITERS = 50
FP64_PEAK_TFLOPS = 37.1  # DMMA m8n8k4 microbenchmark on B200, profiles/r01_fp64_peak_microbench.txt
L2_FLUSH_BYTES = 256 << 20


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            pass
    return {"hbm_gbs": 6650.0, "_source": "fallback (B200_PROFILING.md)"}


def pageable_upload_rates(cpd, ctx, f32: bool, nbytes: int = 2 << 30) -> dict:
    """H2D rate of cpdgpu_tensor_update from PAGEABLE host memory (what a caller holding the
    reference's std::vector-backed DenseTensor passes): the library's staged copy (pinned
    buffers filled by host threads) against a plain cudaMemcpy (CPDGPU_STAGED_UPLOAD=0),
    on a 2 GiB sample.  The headline e2e above uses pinned memory, as the contract asks."""
    n = nbytes // (4 if f32 else 8)
    src = np.ones(n, dtype=np.float32 if f32 else np.float64)  # pageable
    t = cpd.DenseTensor.generate([n // 1024, 1024], cpd.DIST_UNIFORM_PM1 if f32 else cpd.DIST_NORMAL, seed=1,
                                 ctx=ctx, dtype=cpd.F32 if f32 else cpd.F64)
    out = {"sample_bytes": int(src.nbytes)}
    try:
        for key, env in (("staged_gbs", "1"), ("plain_gbs", "0")):
            os.environ["CPDGPU_STAGED_UPLOAD"] = env
            best = 0.0
            for _ in range(3):
                t0 = time.perf_counter()
                t.update(src.ctypes.data)
                ctx.synchronize()
                best = max(best, src.nbytes / (time.perf_counter() - t0) / 1e9)
            out[key] = best
    finally:
        os.environ.pop("CPDGPU_STAGED_UPLOAD", None)
        t.free()
    return out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the GPU is busy."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
            except ValueError:
                continue
            mx = m
            sm.append(s)
            try:
                pw.append(float(parts[2]))
            except ValueError:
                pass
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        busy = [s for s in sm if s > 500] or sm
        return {"sm_mhz": float(np.median(busy)) if busy else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w": float(np.median(pw)) if pw else None}


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def device_normal(ctx, seed, rows, R):
    """Factor matrix drawn by the product's device generator (N(0,1), counter-based)."""
    import paper_1204_1586_b200 as cpd
    t = cpd.DenseTensor.generate([rows, R], cpd.DIST_NORMAL, seed=seed, ctx=ctx)
    v = t.values().reshape(rows, R, order="F")
    t.free()
    return np.asfortranarray(v)


# ---------------------------------------------------------------------------- reference arm

def run_reference(args, cfg):
    """--impl reference: the reference's own cp_gradient_all on this host's cores
    (oracle/_ref, compiled from its sources; the C port if that build is absent),
    each step one bounded sample of the workload (cpu_gradient_sample)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    dims, R, dtype, desc = cfg
    steps = max(1, min(args.steps, 5))
    cpu = cpu_gradient_sample(args, cfg, steps=steps, warmup=min(args.warmup, 1))
    line = {
        "impl": "reference", "metric": f"all-mode CP gradient throughput ({desc})", "value": cpu["value"],
        "unit": "GB/s", "n_gpus": 1, "steps": cpu["steps"], "warmup": min(args.warmup, 1),
        "ms_per_step": cpu["ms_per_step"], "higher_is_better": True,
        "scaling": "strong" if args.config in STRONG_CONFIGS else "weak", "vs_baseline": None, "dtype": dtype,
        "data": "synthetic, counter-based generator", "config": {"workload": args.config, "dims": dims, "R": R},
        "cpu_baseline": cpu,
        "e2e": {"value": cpu["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- our arm

def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_1204_1586_b200 as cpd
    from paper_1204_1586_b200 import build as B
    from paper_1204_1586_b200 import sharded

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and args.gpus != 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    if rank == 0:
        B.build()
    # BENCH_FUNCTIONAL_1GPU=1: functional check of the N>1 code path on a one-GPU box
    # (every rank on device 0, gloo collectives through the host) — never a timing
    functional = os.environ.get("BENCH_FUNCTIONAL_1GPU") == "1"
    if functional:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if functional:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        dist.barrier()
    B.build()  # no-op after rank 0 built it; loads the in-tree .so
    dims, R, dtype, desc = cfg
    N = len(dims)
    ctx = cpd.Context(local)
    stream = torch.cuda.Stream(dev)  # a real stream handle (the legacy default is 0)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)

    f32 = dtype == "f32"
    esize = 4 if f32 else 8
    strong = args.config in STRONG_CONFIGS
    # weak: global dims[:-1] x (dims[-1] * world), every rank one dims-sized slab;
    # strong: the global tensor is dims, each rank a contiguous last-mode slab
    gdims = list(dims) if strong else list(dims[:-1]) + [dims[-1] * world]
    plan = sharded.make_plan(gdims, R, rank, world) if world > 1 else None
    a0, a1 = plan.bounds if plan else (0, gdims[-1])
    ldims = list(gdims[:-1]) + [a1 - a0]
    slab = int(np.prod(ldims))
    y = cpd.DenseTensor.generate(ldims, cpd.DIST_UNIFORM_PM1 if f32 else cpd.DIST_NORMAL, seed=1, ctx=ctx,
                                 offset=a0 * int(np.prod(gdims[:-1])), dtype=cpd.F32 if f32 else cpd.F64)
    gfac = [device_normal(ctx, 100 + k, d, R) for k, d in enumerate(gdims)]
    if plan:
        packed = sharded.pack_local_factors(plan, gfac, np)
        pivot = plan.pivot
    else:
        packed = np.concatenate([f.reshape(-1, order="F") for f in gfac])
        pivot = 0
    fdev = torch.from_numpy(packed).to(dev)
    gdev = torch.zeros_like(fdev)
    flush_needed = slab * esize < 4 * L2_FLUSH_BYTES  # inputs larger than L2 need no flush
    flush = torch.empty(L2_FLUSH_BYTES if flush_needed else 16, dtype=torch.uint8, device=dev)

    # N > 1: the exchange runs inside libcpdgpu.so (cpdgpu_cp_gradient_all_sharded_device:
    # the slab's gradient at the global pivot, then ONE in-place all-reduce of
    # [partial G(1..N-1) | G(N) rows at the slab offset] on the context stream over
    # NCCL; a gloo host all-reduce in the one-GPU functional mode)
    comm = sharded.library_comm(ctx, dist) if plan else None
    gout = torch.zeros(sum(gdims) * R, dtype=torch.float64, device=dev) if plan else gdev

    def step():
        if plan:
            cpd.cp_gradient_all_sharded_device(y, gdims, R, fdev.data_ptr(), gout.data_ptr())
        else:
            cpd.cp_gradient_all_device(y, R, fdev.data_ptr(), gdev.data_ptr(), pivot)

    for _ in range(max(args.warmup, 3)):
        flush.zero_()
        step()
    torch.cuda.synchronize(dev)

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    stops = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = ctx.launch_count()
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            step()
            stops[i].record(stream)
        torch.cuda.synchronize(dev)
        gpu_launches = ctx.launch_count() - launches0  # kernels of the K timed steps
        if world > 1:
            dist.barrier()
        # clocks need a busy window long enough to sample: keep the slab's
        # gradient running for ~1 s after the timed region when the region was
        # short (no collective here: the ranks may loop a different number of times)
        t_end = time.time() + 1.0
        while time.time() < t_end and len(clk.lines) < 10:
            for _ in range(50):
                cpd.cp_gradient_all_device(y, R, fdev.data_ptr(), gdev.data_ptr(), pivot)
            torch.cuda.synchronize(dev)
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, stops)]
    tot_ms = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([tot_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    ms = tot_ms / args.steps
    total_bytes = int(np.prod(gdims)) * esize
    value = total_bytes / (ms * 1e-3) / 1e9

    # dominant kernel: K1 seed contraction, timed live with CUDA events
    ctx.set_timing(True)
    seed_ms = []
    for _ in range(max(10, min(args.steps, 50))):
        flush.zero_()
        cpd.cp_gradient_all_device(y, R, fdev.data_ptr(), gdev.data_ptr(), pivot)
        seed_ms.append(ctx.last_seed_ms())
    ctx.set_timing(False)
    seed_avg = float(np.mean(seed_ms))
    flops = 4.0 * R * slab
    bytes_alg = esize * slab + 2 * 8.0 * R * sum(ldims)
    peaks = measured_peaks()
    tflops = flops / (seed_avg * 1e-3) / 1e12
    hbm_gbs = bytes_alg / (seed_avg * 1e-3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / f"ncu_seed_{args.config}.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    if f32:  # tcgen05 kind::f16 split-fp16 seeds: HBM-bound
        hbm_peak = peaks.get("hbm_gbs", 6539.9)
        path = ctx.last_seed_path()
        kname = {4: "seed_f32i_kernel (K1, tcgen05 kind::f16 on the tensor's fp16 hi/lo operand image, "
                    "both seeds in one pass)",
                 3: "seed_f32f_kernel (K1, tcgen05 kind::f16, fp32 split to hi/lo in the kernel, both seeds "
                    "in one pass)"}.get(path, "seed_f32_kernel<0>+<1> (K1, tcgen05 kind::f16 split-fp16, two passes)")
        roofline = {"bound": "hbm", "achieved": hbm_gbs, "peak": hbm_peak, "unit": "GB/s",
                    "frac": hbm_gbs / hbm_peak, "traffic": traffic,
                    "kernel": kname,
                    "kernel_ms": seed_avg, "algorithmic_flops": flops, "algorithmic_bytes": bytes_alg,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback",
                    "tensor": {"executed_flops": 3 * flops, "achieved_tflops": 3 * tflops,
                               "note": "3 fp16 MMAs per product (hi*hi + lo*hi + hi*lo)"}}
    elif ctx.last_seed_path() == 1:  # both seeds in one pass on the int8 tensor cores (default for c2, c3)
        hbm_peak = peaks.get("hbm_gbs", 6539.9)
        roofline = {"bound": "hbm", "achieved": hbm_gbs, "peak": hbm_peak, "unit": "GB/s",
                    "frac": hbm_gbs / hbm_peak, "traffic": traffic,
                    "kernel": "seed_i8_kernel (K1, fp64 as 6 base-256 digits, tcgen05 kind::i8, both seeds in one pass)",
                    "kernel_ms": seed_avg, "algorithmic_flops": flops, "algorithmic_bytes": bytes_alg,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback",
                    "tensor": {"executed_int8_macs": 21 * flops / 2 * (16 if R <= 16 else 32) / R,
                               "note": "21 digit-pair products per fp64 product, rank padded to the MMA block"}}
    else:  # the binding roof is the slower ideal: bytes / HBM peak vs flops / FP64 DMMA peak
        hbm_peak = peaks.get("hbm_gbs", 6539.9)
        fp64 = {"achieved": tflops, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": tflops / FP64_PEAK_TFLOPS,
                "peak_source": "FP64 DMMA peak measured on B200 (profiles/r01_fp64_peak_microbench.txt)"}
        hbm = {"achieved": hbm_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": hbm_gbs / hbm_peak,
               "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"}
        hbm_bound = bytes_alg / (hbm_peak * 1e9) > flops / (FP64_PEAK_TFLOPS * 1e12)
        main, other = (hbm, fp64) if hbm_bound else (fp64, hbm)
        roofline = {"bound": "hbm" if hbm_bound else "tensor", **{k: main[k] for k in ("achieved", "peak", "unit", "frac")},
                    "traffic": traffic, "kernel": "seed_f64_kernel (K1, fp64 DMMA, both seeds in one pass)",
                    "kernel_ms": seed_avg, "algorithmic_flops": flops, "algorithmic_bytes": bytes_alg,
                    "peak_source": main["peak_source"], ("tensor" if hbm_bound else "hbm"): other}

    # the paper's comparison (Algorithm 1 vs 2): N direct mode-n MTTKRPs, one pass over Y each
    alg1 = None
    if world == 1 and not args.no_alg1:
        reps = 3
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
        for i in range(reps + 1):
            if i:
                flush.zero_()
                ev[2 * (i - 1)].record(stream)
            for n in range(1, N + 1):
                cpd.mttkrp_direct_device(y, R, fdev.data_ptr(), gdev.data_ptr(), n)
            if i:
                ev[2 * (i - 1) + 1].record(stream)
        torch.cuda.synchronize(dev)
        a_ms = float(np.mean([ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(reps)]))
        alg1 = {"ms_per_step": a_ms, "rho": a_ms / ms,
                "what": f"all-mode gradient as {N} direct mode-n MTTKRPs (mttkrp_direct, one pass over Y each) "
                        "on the same device, same inputs; rho = Algorithm 1 time / Algorithm 2 time"}

    # e2e through the host C-ABI: H2D of Y from pinned memory + factors, D2H of gradients
    e2e = None
    if not args.no_e2e and world == 1 and host_memory_ok(3 * slab * esize):
        host_y = torch.empty(slab, dtype=torch.float32 if f32 else torch.float64).pin_memory()
        host_y.copy_(torch.from_numpy(y.values()))
        facs = [f.copy(order="F") for f in gfac]
        e_steps = max(3, min(args.steps, 20 if slab * esize < (1 << 30) else 3))
        for _ in range(2):
            y.update(host_y.data_ptr())
            cpd.cp_gradient_all(y, facs)
        torch.cuda.synchronize(dev)
        t_up = t_grad = 0.0
        t0 = time.perf_counter()
        for _ in range(e_steps):
            ta = time.perf_counter()
            y.update(host_y.data_ptr())
            ctx.synchronize()  # (the stream serialises the two anyway; this only splits the time)
            tb = time.perf_counter()
            cpd.cp_gradient_all(y, facs)
            t_up += tb - ta
            t_grad += time.perf_counter() - tb
        dt = (time.perf_counter() - t0) / e_steps
        e2e = {"value": slab * esize / dt / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": slab * esize + 8 * R * sum(dims),
               "d2h_bytes_per_step": 8 * R * sum(dims), "ms_per_step": dt * 1e3,
               "update_ms": t_up / e_steps * 1e3, "gradient_call_ms": t_grad / e_steps * 1e3,
               "timing": "wall clock around synchronous host-API calls: update = H2D of Y from pinned memory "
                         "(cpdgpu_tensor_update), gradient call = factors in, per-tensor-version scale record, "
                         "gradient, gradients out"}

        e2e["pageable_upload"] = pageable_upload_rates(cpd, ctx, f32)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, cfg, y if f32 else None)

    if rank == 0:
        line = {
            "metric": f"all-mode CP gradient throughput ({desc})", "value": value, "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": dtype,
            "data": ("synthetic U(-1,1) fp32 tensor, N(0,1) factors" if f32 else "synthetic N(0,1)")
                    + ", counter-based generator",
            "config": {"workload": args.config, "dims": dims, "R": R, "local_dims": ldims,
                       "global_dims": gdims, "parallelism": f"slab{world}" if world > 1 else "single",
                       "l2": ("flushed before every step (256 MiB memset outside the events)" if flush_needed
                              else "inputs larger than L2 (no flush)")},
            "gpu_launches": gpu_launches, "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu,
            "algorithm1_direct": alg1, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def host_memory_ok(nbytes):
    try:
        import psutil
        return psutil.virtual_memory().available > nbytes
    except Exception:
        return False


def reference_build():
    """oracle/ref.py when the reference itself is built (oracle/_ref), else None."""
    sys.path.insert(0, str(ROOT / "oracle"))
    try:
        import ref
        if (ROOT / "oracle" / "_ref" / "libcpdref.so").exists():
            ref.load()
            return ref
    except Exception as e:  # noqa: BLE001 - fall back to the port, say why
        print(f"reference build unavailable ({e}); timing the C port", file=sys.stderr)
    return None


def cpu_gradient_sample(args, cfg, steps=None, warmup=1):
    """CPU time of the workload's all-mode gradient on a bounded sample, on this
    host's cores.  Preferred: the reference ITSELF (oracle/_ref: its own
    mttkrp.cpp / Eigen code path compiled with its Release flags, Eigen replaced
    by oracle/shim), which is single-threaded, run as one independent reference
    call per core on mode-1 slabs of the tensor (the gradients of the slabs sum
    exactly: the same decomposition the GPUs shard by).  fp64 configs: the full
    tensor; c5 (300^4, 32 GB fp32 — beyond this host's memory in fp64): a
    (cores x 300 x 300 x 300) tensor of the same U(-1,1) fp32 values upcast to
    fp64 (the reference is fp64-only), same R and pivot structure, reported per
    fp32 tensor byte like the GPU arm.  Fallback: the OpenMP C port."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O
    dims, R, dtype, desc = cfg
    cores = host_cores()
    esize = 4 if dtype == "f32" else 8
    ref = reference_build()
    if dtype == "f32":
        sd = [cores] + list(dims[1:])
        n = int(np.prod(sd))
        y = O.fill_upm1_f32(1, n, nthreads=cores).astype(np.float64)
    else:
        sd = list(dims)
        n = int(np.prod(sd))
        y = O.fill_normal(1, n, nthreads=cores)
    f = [O.fill_normal(100 + k, d * R).reshape(d, R, order="F") for k, d in enumerate(sd)]
    single = None
    if ref is not None:
        # single-core figure: the reference as built, one thread,
        # one call on the whole fp64 tensor (c5: one 300^3 slab of the sample)
        if dtype == "f32":
            sd1 = [1] + list(sd[1:])
            y1 = np.ascontiguousarray(y.reshape(sd, order="F")[:1].reshape(-1, order="F"))
            f1 = [np.asfortranarray(f[0][:1])] + f[1:]
        else:
            sd1, y1, f1 = sd, y, f
        t1 = ref.Tensor(y1, sd1, parts=1)
        if y1.size * 8 <= (256 << 20):
            t1.cp_gradient_all(f1)
        s1 = t1.time_cp_gradient_all(f1, 1)
        t1.close()
        del y1
        single = {"value": int(np.prod(sd1)) * esize / s1 / 1e9, "unit": "GB/s", "cores": 1,
                  "ms_per_step": s1 * 1e3,
                  "sample": f"one call of the reference's cp_gradient_all on the {'x'.join(map(str, sd1))} fp64 "
                            "tensor, one thread"}
        t = ref.Tensor(y, sd, parts=min(cores, sd[0]), axis=0)
        del y
        for _ in range(warmup):
            t.cp_gradient_all(f)
        first = t.time_cp_gradient_all(f, 1)
        reps = steps or max(1, int(args.cpu_seconds / max(first, 1e-6)))
        dt = t.time_cp_gradient_all(f, reps) if reps > 1 else first
        t.close()
        kind, threads = "reference", min(cores, sd[0])
        how = (f"the reference's own cp_gradient_all (oracle/_ref: /root/reference/proj/core built -O3 -DNDEBUG, "
               f"Eigen shim), one single-threaded call per core on {threads} mode-1 slabs")
    else:
        t0 = time.perf_counter()
        reps = 0
        while reps < (steps or 10 ** 9):
            O.cp_gradient_all(y, sd, f, nthreads=cores)
            reps += 1
            if not steps and time.perf_counter() - t0 > args.cpu_seconds:
                break
        dt = (time.perf_counter() - t0) / reps
        kind, threads, how = "port", cores, "oracle/cpd_oracle.c (the C port), OpenMP"
    what = "full" if sd == list(dims) else f"{'x'.join(map(str, sd))} sample ({dtype} values upcast to fp64) of the"
    return {"value": n * esize / dt / 1e9, "unit": "GB/s", "cores": threads, "kind": kind,
            "sample": f"{reps} x {what} {args.config} gradient, {how}", "ms_per_step": dt * 1e3, "steps": reps,
            "host_cores": cores, "single_core": single}


def cpu_baseline(args, cfg, ydev=None):
    return cpu_gradient_sample(args, cfg)


# ---------------------------------------------------------------------------- CP_ALS (c4)

def c4_truth(I, R, N, seed, fill):
    """Factors of the rank-R N(0,1) ground-truth model and of the init (separate seed)."""
    truth = [fill(seed * 100 + k, I * R).reshape(I, R, order="F") for k in range(N)]
    init = [fill(seed * 1000 + 7 + k, I * R).reshape(I, R, order="F") for k in range(N)]
    return truth, init


def c4_device_tensor(ctx, dims, truth, seed=4):
    """Y = sigma E + full(model), sigma = |full| / (10 |E|) (SNR 20 dB), built on the device."""
    import paper_1204_1586_b200 as cpd
    y = cpd.DenseTensor.generate(dims, cpd.DIST_NORMAL, seed=seed, ctx=ctx)
    e2 = y.norm2()
    t = cpd.DenseTensor.generate(dims, cpd.DIST_NORMAL, seed=seed, ctx=ctx)
    t.axpby_kruskal(0.0, 1.0, truth)
    full2 = t.norm2()
    t.free()
    y.axpby_kruskal(float(np.sqrt(full2) / (10.0 * np.sqrt(e2))), 1.0, truth)
    return y


def c4_slab_tensor(ctx, dims, truth, lo, hi, allsum, seed=4):
    """Rows [lo, hi) of the last mode of c4_device_tensor's Y (the same counter-based
    noise and model; the noise scale from the global norms via `allsum`)."""
    import paper_1204_1586_b200 as cpd
    ldims = list(dims[:-1]) + [hi - lo]
    off = lo * int(np.prod(dims[:-1]))
    ltruth = list(truth[:-1]) + [np.asfortranarray(truth[-1][lo:hi])]
    y = cpd.DenseTensor.generate(ldims, cpd.DIST_NORMAL, seed=seed, ctx=ctx, offset=off)
    e2 = allsum(y.norm2())
    t = cpd.DenseTensor.generate(ldims, cpd.DIST_NORMAL, seed=seed, ctx=ctx, offset=off)
    t.axpby_kruskal(0.0, 1.0, ltruth)
    full2 = allsum(t.norm2())
    t.free()
    y.axpby_kruskal(float(np.sqrt(full2) / (10.0 * np.sqrt(e2))), 1.0, ltruth)
    return y


def als_metric(desc):
    return f"CP_ALS iterations per second ({desc})"


def cpu_als_sample(args, yh, dims, init, max_sweeps=None):
    """CPU fast ALS sweeps of the c4 tensor: the reference itself (oracle/_ref,
    cpd::als_sweep_fast: single-threaded, a Gauss-Seidel sweep has no slab
    parallelism) or, without that build, the OpenMP C port."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O
    cores = host_cores()
    f = [a.copy(order="F") for a in init]
    ref = reference_build()
    done, spent = 0, 0.0
    limit = max_sweeps or 10 ** 9
    if ref is not None:
        t = ref.Tensor(yh, dims)
        while done < limit and (done < 1 or spent < args.cpu_seconds):
            _, sec = t.als_sweep_fast(f)
            spent += sec
            done += 1
        t.close()
        kind, threads, how = "reference", 1, ("the reference's own cpd::als_sweep_fast (oracle/_ref: "
                                              "/root/reference/proj/core built -O3 -DNDEBUG, Eigen shim), 1 thread")
    else:
        t0 = time.perf_counter()
        while done < limit and (done < 1 or time.perf_counter() - t0 < args.cpu_seconds):
            O.als_sweep_fast(yh, dims, f, nthreads=cores)
            done += 1
        spent = time.perf_counter() - t0
        kind, threads, how = "port", cores, "oracle/cpd_oracle.c (the C port), OpenMP"
    dt = spent / done
    return {"value": 1.0 / dt, "unit": "iters/s", "cores": threads, "kind": kind,
            "sample": f"{done} fast ALS sweeps of the full {args.config} tensor, {how}", "ms_per_step": dt * 1e3,
            "steps": done, "host_cores": cores}


def run_reference_als(args, cfg):
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    dims, R, dtype, desc = cfg
    cores = host_cores()
    n = int(np.prod(dims))
    truth, init = c4_truth(dims[0], R, len(dims), 4, O.fill_normal)
    e = O.fill_normal(4, n, nthreads=cores)
    full = O.full(dims, truth)
    sigma = float(np.sqrt(np.dot(full, full)) / (10.0 * np.sqrt(np.dot(e, e))))
    y = sigma * e + full
    del e, full
    cpu = cpu_als_sample(args, y, dims, init, max_sweeps=max(1, min(args.steps, 3)))
    del y
    dt = cpu["ms_per_step"] * 1e-3
    line = {
        "impl": "reference", "metric": als_metric(desc), "value": 1.0 / dt, "unit": "iters/s", "n_gpus": 1,
        "steps": cpu["steps"], "warmup": 0, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic rank-16 N(0,1) model + N(0,1) noise at 20 dB, counter-based generator",
        "config": {"workload": args.config, "dims": dims, "R": R},
        "cpu_baseline": cpu,
        "e2e": {"value": 1.0 / dt, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours_als(args, cfg):
    """c4: K fast ALS sweeps on the device (cpdgpu_als_run), per-sweep CUDA events
    on the launching stream.  Y (6.2 GB) is far larger than L2.  N>1 shards the
    last mode (cpdgpu_als_run_sharded: the global Gauss-Seidel order, an all-reduce
    of each G(n), n < N, before its update; strong scaling)."""
    import torch
    import torch.distributed as dist

    import paper_1204_1586_b200 as cpd
    from paper_1204_1586_b200 import build as B
    from paper_1204_1586_b200 import sharded

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if rank == 0:
        B.build()
    # BENCH_FUNCTIONAL_1GPU=1: functional check of the N>1 code path on a one-GPU box
    # (every rank on device 0, gloo collectives through the host) — never a timing
    functional = os.environ.get("BENCH_FUNCTIONAL_1GPU") == "1"
    if functional:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if functional:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        dist.barrier()
    B.build()
    dims, R, dtype, desc = cfg
    N = len(dims)
    esize = 8
    ctx = cpd.Context(local)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    truth, init = c4_truth(dims[0], R, N, 4, lambda s, n: device_normal(ctx, s, n, 1).reshape(-1))
    if world > 1:
        lo, hi = cpd.slab_bounds(dims[-1], world, rank)

        def allsum(v):
            t = torch.tensor([v], device=dev, dtype=torch.float64)
            dist.all_reduce(t)
            return float(t.item())

        y = c4_slab_tensor(ctx, dims, truth, lo, hi, allsum)
        loc_init = list(init[:-1]) + [init[-1][lo:hi]]
        comm = sharded.library_comm(ctx, dist)

        def run_sweeps(k):
            return cpd.als_run_sharded(y, dims, [f.copy(order="F") for f in init], max_iters=k)
    else:
        y = c4_device_tensor(ctx, dims, truth)
        loc_init = init
        comm = None

        def run_sweeps(k):
            return cpd.run(y, init, cpd.SolveOptions(max_iters=k)).trace
    slab = int(np.prod(y.dims))

    run_sweeps(max(args.warmup, 3))  # warm-up (graph capture)
    torch.cuda.synchronize(dev)
    launches0 = ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        trace = run_sweeps(args.steps)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        gpu_launches = ctx.launch_count() - launches0
        if world > 1:
            dist.barrier()
            for _ in range(2):  # a fixed count: every rank runs the same collectives
                run_sweeps(20)
        else:
            t_end = time.time() + 2.0  # keep the same sweep busy until the sampler has seen it
            while time.time() < t_end and len(clk.lines) < 10:
                run_sweeps(20)
    sweep_s = float(np.sum(trace.seconds))
    if world > 1:
        t = torch.tensor([sweep_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sweep_s = float(t.item())
        comm.close()
    ms = sweep_s / args.steps * 1e3
    value = args.steps / sweep_s

    # dominant kernels: the two seed passes of a sweep (K1 right pass, then the
    # column-block left pass after the right phase's updates), CUDA events around
    # each launch on the launching stream (ctx timing mode runs the sweep eagerly)
    ctx.set_timing(True)
    seed_ms = []
    f_h = [np.array(f, dtype=np.float64, order="F", copy=True) for f in loc_init]
    for _ in range(6):  # N > 1: the slab's own (local) sweep, whose seeds are the sharded sweep's
        cpd.als_sweep_fast(y, f_h)
        seed_ms.append(ctx.last_seed_ms())
    ctx.set_timing(False)
    seed_avg = float(np.mean(seed_ms[1:]))
    flops = 4.0 * R * slab
    bytes_sweep = 2.0 * 8.0 * slab  # two reads of Y per Gauss-Seidel sweep (mandatory)
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6539.9)
    tflops = flops / (seed_avg * 1e-3) / 1e12
    hbm_gbs = bytes_sweep / (seed_avg * 1e-3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / f"ncu_seed_{args.config}.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": hbm_gbs, "peak": hbm_peak, "unit": "GB/s",
                "frac": hbm_gbs / hbm_peak, "traffic": traffic,
                "kernel": "seed_f64_kernel<NT,1> right pass + seed_left_cols_kernel left pass (the 2 Y reads of one sweep)",
                "kernel_ms": seed_avg, "algorithmic_bytes": bytes_sweep, "algorithmic_flops": flops,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "tensor": {"achieved": tflops, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                           "frac": tflops / FP64_PEAK_TFLOPS,
                           "peak_source": "FP64 DMMA peak measured on B200 (profiles/r01_fp64_peak_microbench.txt)"}}

    # e2e: a full run() through the host API with Y uploaded from pinned host memory
    e2e = None
    if not args.no_e2e and world == 1 and host_memory_ok(3 * slab * esize):
        host_y = torch.empty(slab, dtype=torch.float64).pin_memory()
        host_y.copy_(torch.from_numpy(y.values()))
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        y.update(host_y.data_ptr())
        r2 = cpd.run(y, init, cpd.SolveOptions(max_iters=C4_ITERS))
        dt = time.perf_counter() - t0
        e2e = {"value": C4_ITERS / dt, "unit": "iters/s",
               "h2d_bytes_per_step": (slab * 8 + 8 * R * sum(dims)) / C4_ITERS,
               "d2h_bytes_per_step": (8 * R * sum(dims) + 8 * 3 * C4_ITERS) / C4_ITERS,
               "ms_per_step": dt * 1e3 / C4_ITERS,
               "timing": f"wall clock around one host-API run(): H2D of Y + {C4_ITERS} sweeps + fit trace + "
                         "factors back, divided by the sweep count",
               "final_rel_error": r2.trace.rel_error[-1]}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        yh = y.values()
        cpu = cpu_als_sample(args, yh, dims, init)
        del yh
    if rank == 0:
        line = {
            "metric": als_metric(desc), "value": value, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic rank-16 N(0,1) model + N(0,1) noise at 20 dB, counter-based generator",
            "config": {"workload": args.config, "dims": dims, "R": R,
                       "parallelism": f"last-mode slabs x{world} (sharded ALS)" if world > 1 else "single",
                       "l2": "inputs larger than L2 (6.2 GB tensor)",
                       "run_ms_incl_fit": ev0.elapsed_time(ev1),
                       "final_rel_error": trace.rel_error[-1]},
            "gpu_launches": gpu_launches, "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=list(CONFIGS), default="c5")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-alg1", action="store_true", help="skip the Algorithm 1 (direct MTTKRP) comparison")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.config in ALS_CONFIGS:
        return run_reference_als(args, cfg) if args.impl == "reference" else run_ours_als(args, cfg)
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
