#!/bin/bash
# c5 fused fp32 seed timing experiments (wrong results): CPDGPU_F32F_KNOBS x CPDGPU_F32_BAND
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-knobs2}
: > $O/${T}.txt
for band in ${BANDS:-3 2}; do
  for k in ${KNOBS:-0 8 64 72}; do
    CPDGPU_F32_BAND=$band CPDGPU_F32F_KNOBS=$k timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('band=$band knobs=$k', round(d['ms_per_step']*1e3,1), 'us  seed', round(r['kernel_ms']*1e3,1), 'mhz', d['clocks']['sm_mhz'])
" >> $O/${T}.txt
  done
done
