#!/bin/bash
# c5 fused fp32 seed: image layout (CPDGPU_F32_IMG_CHUNK) x knobs (0 full, 32 no MMAs: the stream alone)
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-knobs3}
: > $O/${T}.txt
for rep in 1 2; do
for ch in 0 1; do
  for k in ${KNOBS:-0 32}; do
    CPDGPU_F32_IMG_CHUNK=$ch CPDGPU_F32F_KNOBS=$k timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('chunk=$ch knobs=$k', round(d['ms_per_step']*1e3,1), 'us  seed', round(r['kernel_ms']*1e3,1), 'mhz', d['clocks']['sm_mhz'])
" >> $O/${T}.txt
  done
done
done
