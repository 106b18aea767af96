import json, sys
for l in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench.txt"):
    try:
        d = json.loads(l)
    except Exception:
        if l.strip(): print("  |", l.rstrip()[:200])
        continue
    r = d.get("roofline") or {}
    print(d["config"]["workload"], "ms/step %.4f" % d["ms_per_step"], "GB/s %.0f" % d["value"],
          "seed_ms %.4f" % r.get("kernel_ms", 0), "TF %.2f" % r.get("achieved", 0),
          "hbm %.0f" % (r.get("hbm") or {}).get("achieved", 0), "launches", d.get("gpu_launches"))
