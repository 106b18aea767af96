#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-f32l0}
timeout 900 python -m pytest tests/test_gpu_f32.py tests/test_gpu_sharded.py tests/test_gpu_sharded_abi.py -q -x -s -p no:cacheprovider > $O/${T}_pytest.txt 2>&1
echo "rc=$?" >> $O/${T}_pytest.txt
: > $O/${T}_ab.txt
for rep in 1 2 3; do
  for v in 0 1; do
    CPDGPU_F32_L0=$v timeout 300 python bench.py --config c5 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('l0=$v', round(d['ms_per_step'],3), 'ms  seed', round(r['kernel_ms'],3), 'mhz', d['clocks']['sm_mhz'])
" >> $O/${T}_ab.txt
  done
done
B="python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1"
if timeout 300 $B > /dev/null 2>&1; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/${T}_launches_c5.csv $B > /dev/null 2>&1
fi
