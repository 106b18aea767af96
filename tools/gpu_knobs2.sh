#!/bin/bash
# c5 seed: which term bounds the MMA issue?  knobs 2 (one right MMA per k-step), 4 (one left
# MMA per k-step), 6 (both), 0 (full), each with the per-warp cycle trace
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-knobs2}
: > $O/${T}.txt
for k in 0 2 4 6 0; do
  echo "knobs=$k" >> $O/${T}.txt
  CPDGPU_F32F_KNOBS=$k timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | python -c '
import sys,json
for l in sys.stdin:
  if l.startswith("{"):
    d=json.loads(l); print("step_ms=%.3f seed_ms=%.3f sm_mhz=%s" % (d["ms_per_step"], d["roofline"]["kernel_ms"], d["clocks"]["sm_mhz"]))
' >> $O/${T}.txt
  CPDGPU_F32F_KNOBS=$k CPDGPU_SEED_TRACE=1 timeout 300 python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | grep trace | tail -1 >> $O/${T}.txt
done
