#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-l0b}
: > $O/${T}_ab.txt
for rep in 1 2; do
  for c in c2 c3; do
    for v in l0a l0b; do
      CPDGPU_ABI_PARTIAL=1 CPDGPU_LIB=tools/bisect_$v.so timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('$v', '$c', round(d['ms_per_step']*1e3,1), 'us  seed', round(r['kernel_ms']*1e3,1))
" >> $O/${T}_ab.txt
    done
  done
done
for v in l0a l0b; do
  CPDGPU_ABI_PARTIAL=1 CPDGPU_LIB=tools/bisect_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:l0_kernel -c 4 --csv --log-file $O/${T}_ncu_c5_$v.csv python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 > /dev/null 2>&1
done
