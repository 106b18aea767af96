#!/bin/bash
# fused fp32 seed (c5) ablation: CPDGPU_F32F_KNOBS timing experiments + the per-warp
# cycle trace (CPDGPU_SEED_TRACE=1); each line is a bench run of the same tensor
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-knobs}
B="python bench.py --config ${CFG:-c5} --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline --no-alg1"
: > $O/${T}.txt
for k in ${KNOBS:-0 8 32 128 256 64 16}; do
  echo "knobs=$k $(CPDGPU_F32F_KNOBS=$k timeout 300 $B 2>&1 | python -c '
import sys,json
for l in sys.stdin:
  if l.startswith("{"):
    d=json.loads(l); print("step_ms=%.3f seed_ms=%.3f sm_mhz=%s" % (d["ms_per_step"], d["roofline"]["kernel_ms"], d["clocks"]["sm_mhz"]))
  elif "error" in l.lower() or "Traceback" in l: print(l.strip())
')" >> $O/${T}.txt
done
CPDGPU_SEED_TRACE=1 timeout 300 python bench.py --config ${CFG:-c5} --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | grep trace | tail -3 >> $O/${T}.txt
