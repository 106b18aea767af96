#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-pad}
timeout 1200 python -m pytest tests/test_gpu_i8.py tests/test_gpu_gradient.py -q -x -p no:cacheprovider > $O/${T}_pytest.txt 2>&1
echo "rc=$?" >> $O/${T}_pytest.txt
: > $O/${T}_ab.txt
for rep in 1 2; do
  for v in 0 1; do
    CPDGPU_I8_PAD=$v timeout 300 python bench.py --config c3 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('pad=$v c3', round(d['ms_per_step']*1e3,1), 'us  seed', round(r['kernel_ms']*1e3,1), 'frac', round(r['frac'],3))
" >> $O/${T}_ab.txt
  done
done
B="python bench.py --config c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"seed_i8|pad_rows" -c 4 --csv --log-file $O/${T}_dram_c3.csv $B > /dev/null 2>&1
