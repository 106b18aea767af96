#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-pair2}
timeout 900 python -m pytest tests/test_gpu_f32.py -q -x -p no:cacheprovider -k "full_c5 or matches" > $O/${T}_pytest.txt 2>&1
echo "rc=$?" >> $O/${T}_pytest.txt
: > $O/${T}_ab.txt
for rep in 1 2; do
  for v in 0 1; do
    CPDGPU_F32_PAIR=$v timeout 300 python bench.py --config c5 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('pair=$v', round(d['ms_per_step'],3), 'ms  seed', round(r['kernel_ms'],3), 'mhz', d['clocks']['sm_mhz'])
" >> $O/${T}_ab.txt
  done
done
CPDGPU_F32_PAIR=1 CPDGPU_SEED_TRACE=1 timeout 300 python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | grep trace | tail -1 >> $O/${T}_ab.txt
