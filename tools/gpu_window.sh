#!/bin/bash
# fused fp32 seed (c5): right-drain window sweep (CPDGPU_F32_WINDOW) and the c5 accuracy test per window
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-window}
B="python bench.py --config c5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1"
: > $O/${T}.txt
for w in ${WINDOWS:-4 8 16 2}; do
  echo "window=$w $(CPDGPU_F32_WINDOW=$w timeout 300 $B 2>&1 | python -c '
import sys,json
for l in sys.stdin:
  if l.startswith("{"):
    d=json.loads(l); print("step_ms=%.3f seed_ms=%.3f sm_mhz=%s" % (d["ms_per_step"], d["roofline"]["kernel_ms"], d["clocks"]["sm_mhz"]))
')" >> $O/${T}.txt
done
for w in ${ACC_WINDOWS:-8 16}; do
  CPDGPU_F32_WINDOW=$w timeout 900 python -m pytest tests/test_gpu_f32.py -q -x -k "full_c5" -s 2>&1 | tail -5 | sed "s/^/acc w=$w: /" >> $O/${T}.txt
done
