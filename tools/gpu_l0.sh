#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-l0}
: > $O/${T}_ab.txt
for rep in 1 2; do
  for c in c2 c3; do
    for v in 1024 512 256 128; do
      CPDGPU_L0_ROWS=$v timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('rows=$v', '$c', round(d['ms_per_step']*1e3,1), 'us  seed', round(r['kernel_ms']*1e3,1))
" >> $O/${T}_ab.txt
    done
  done
done
for v in 1024 256; do
  CPDGPU_L0_ROWS=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:l0_kernel -c 6 --csv --log-file $O/${T}_ncu_$v.csv python bench.py --config c2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 > /dev/null 2>&1
done
