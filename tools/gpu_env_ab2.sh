#!/bin/bash
# A/B of environment settings on one config (same build); each setting is a
# space-free "VAR=val,VAR2=val" string:
#   SETTINGS="CPDGPU_F32_IMG_CHUNK=0 CPDGPU_F32_IMG_CHUNK=1,CPDGPU_F32F_KNOBS=32" CONFIG=c5 REPS=2 TAG=x bash tools/gpu_env_ab2.sh
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-envab2}
: > $O/${T}_ab.txt
for rep in $(seq ${REPS:-2}); do
  for st in ${SETTINGS}; do
    env ${st//,/ } timeout 300 python bench.py --config ${CONFIG:-c5} --steps ${STEPS:-20} --warmup 5 --no-e2e --no-cpu-baseline --no-alg1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('$st', d['config']['workload'], round(d['ms_per_step']*1e3,1), 'us  seed', round(r['kernel_ms']*1e3,1), 'mhz', d['clocks']['sm_mhz'], d['clocks'].get('power_w'))
" >> $O/${T}_ab.txt
  done
done
