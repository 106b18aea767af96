#!/bin/bash
# A/B of prebuilt variants on c5 with the seed cycle trace
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-abt}
: > $O/${T}_ab.txt
for rep in 1 2; do
  for v in ${VARIANTS}; do
    CPDGPU_ABI_PARTIAL=1 CPDGPU_LIB=tools/bisect_$v.so timeout 300 python bench.py --config c5 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('$v', round(d['ms_per_step'],3), 'ms  seed', round(r['kernel_ms'],3), 'mhz', d['clocks']['sm_mhz'])
" >> $O/${T}_ab.txt
  done
done
for v in ${VARIANTS}; do
  echo "$v" >> $O/${T}_ab.txt
  CPDGPU_ABI_PARTIAL=1 CPDGPU_LIB=tools/bisect_$v.so CPDGPU_SEED_TRACE=1 timeout 300 python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | grep trace | tail -1 >> $O/${T}_ab.txt
done
