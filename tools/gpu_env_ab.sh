#!/bin/bash
# A/B of an environment switch on one config (same build):
#   ENVVAR=CPDGPU_I8 VALUES="0 1" CONFIG=c1 REPS=2 STEPS=50 TAG=x bash tools/gpu_env_ab.sh
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-envab}
: > $O/${T}_ab.txt
for rep in $(seq ${REPS:-2}); do
  for v in ${VALUES}; do
    env ${ENVVAR}=$v timeout 300 python bench.py --config ${CONFIG:-c5} --steps ${STEPS:-20} --warmup 5 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('${ENVVAR}=$v', d['config']['workload'], round(d['ms_per_step']*1e3,1), 'us  seed', round(r['kernel_ms']*1e3,1), 'mhz', d['clocks']['sm_mhz'])
" >> $O/${T}_ab.txt
  done
done
