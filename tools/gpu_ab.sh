#!/bin/bash
# A/B step and seed timing of prebuilt variants (tools/bisect_<v>.so) on one box:
#   VARIANTS="a b" CONFIGS="c2 c3" REPS=2 TAG=x bash tools/gpu_ab.sh
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-ab}
: > $O/${T}_ab.txt
for rep in $(seq ${REPS:-2}); do
  for c in ${CONFIGS:-c2}; do
    for v in ${VARIANTS}; do
      CPDGPU_ABI_PARTIAL=1 CPDGPU_LIB=tools/bisect_$v.so timeout 300 python bench.py --config $c --steps ${STEPS:-50} --warmup 5 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('$v', '$c', round(d['ms_per_step']*1e3,1), 'us  seed', round(r['kernel_ms']*1e3,1), 'mhz', d['clocks']['sm_mhz'])
" >> $O/${T}_ab.txt
    done
  done
done
