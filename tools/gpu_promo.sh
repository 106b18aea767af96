#!/bin/bash
# int8 pass: L2 promotion of the Y boxes (CPDGPU_I8_PROMO) on c2 and c3, and DRAM bytes per seed
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-promo}
: > $O/${T}_ab.txt
for rep in 1 2; do
  for c in c3 c2; do
    for v in 256 128 64 0; do
      CPDGPU_I8_PROMO=$v timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('promo=$v', '$c', round(d['ms_per_step']*1e3,1), 'us  seed', round(r['kernel_ms']*1e3,1))
" >> $O/${T}_ab.txt
    done
  done
done
for v in 256 64 0; do
  B="python bench.py --config c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1"
  CPDGPU_I8_PROMO=$v timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:seed_i8 -c 3 --csv --log-file $O/${T}_dram_c3_$v.csv $B > /dev/null 2>&1
done
