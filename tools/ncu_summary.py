"""Summarise an ncu --set full report into profiles/ncu_seed_<cfg>.json (units
normalised: us, bytes, Hz).  dram_bytes_per_launch = read + write bytes summed
over the listed kernels (one gradient, or one ALS sweep's two passes), which
bench.py reports as roofline.traffic.

  python tools/ncu_summary.py <report.ncu-rep> <cfg> <algorithmic_bytes> "<label>"
"""
import csv, json, subprocess, sys
from pathlib import Path

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1,
         "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u = r[0], r[1]
    return [{k: (v, un) for k, v, un in zip(h, x, u)} for x in r[2:]]


def val(d, k):
    if k not in d:
        return None
    v, u = d[k]
    try:
        return float(v.replace(",", "")) * SCALE.get(u, 1)
    except ValueError:
        return None


def main(rep, cfg, algo_bytes, label):
    ks = []
    for d in rows(rep):
        rd, wr = val(d, "dram__bytes_read.sum"), val(d, "dram__bytes_write.sum")
        ks.append({"kernel": d["Kernel Name"][0][:80], "gpu_time_us": val(d, "gpu__time_duration.sum"),
                   "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": (rd or 0) + (wr or 0),
                   "registers_per_thread": val(d, "launch__registers_per_thread"),
                   "dmma_pipe_active_pct_active": val(d, "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
                   "tensor_pipe_active_pct_active": val(d, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                   "issue_active_pct": val(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                   "smem_bank_conflicts": val(d, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
                   "sm_clock_hz": val(d, "gpc__cycles_elapsed.avg.per_second")})
    out = {"source": f"ncu --set full --import-source on --clock-control none, {Path(rep).name}",
           "label": label, "algorithmic_bytes_per_launch": algo_bytes, "kernels": ks,
           "dram_bytes_per_launch": sum(k["traffic_bytes"] for k in ks),
           "dram_bytes_note": "dram__bytes_read.sum + dram__bytes_write.sum over the listed kernels, read by bench.py "
                              "as roofline.traffic"}
    dst = Path(__file__).resolve().parent.parent / "profiles" / f"ncu_seed_{cfg}.json"
    dst.write_text(json.dumps(out, indent=1))
    print(dst, out["dram_bytes_per_launch"])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], float(sys.argv[3]), sys.argv[4])
