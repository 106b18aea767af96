#!/bin/bash
# CTA-pair (cluster of 2, DSMEM) left-partial reduction of the fused fp32 pass:
# parity (fp32 tests incl. c5 full size, sharded slabs, watchdog), then A/B of
# CPDGPU_F32_PAIR=0/1 on the same build
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-pair}
timeout 900 python -m pytest tests/test_gpu_f32.py tests/test_gpu_sharded.py tests/test_gpu_watchdog.py -q -x -s -p no:cacheprovider > $O/${T}_pytest.txt 2>&1
echo "rc=$?" >> $O/${T}_pytest.txt
: > $O/${T}_ab.txt
for rep in 1 2 3; do
  for v in 0 1; do
    CPDGPU_F32_PAIR=$v timeout 300 python bench.py --config c5 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('pair=$v', round(d['ms_per_step'],3), 'ms  seed', round(r['kernel_ms'],3), 'mhz', d['clocks']['sm_mhz'])
  elif 'rror' in l: print(l.strip()[:300])
" >> $O/${T}_ab.txt
  done
done
B="python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1"
if timeout 300 $B > /dev/null 2>&1; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/${T}_launches_c5.csv $B > /dev/null 2>&1
fi
