#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-ab6}
timeout 600 python -m pytest tests/test_gpu_i8.py -q -p no:cacheprovider > $O/${T}_pytest.txt 2>&1
echo "rc=$?" >> $O/${T}_pytest.txt
: > $O/${T}_ab.txt
for rep in 1 2; do
  for v in ${VARIANTS:-old p1 p2 p4 p8}; do
    CPDGPU_LIB=tools/bisect_$v.so timeout 300 python bench.py --config c5 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('$v', round(d['ms_per_step'],3), 'ms  seed', round(r['kernel_ms'],3), 'mhz', d['clocks']['sm_mhz'])
" >> $O/${T}_ab.txt
  done
done
