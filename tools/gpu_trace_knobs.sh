#!/bin/bash
# Fused fp32 seed per-role cycle trace (CPDGPU_SEED_TRACE) under timing-experiment
# knobs (CPDGPU_F32F_KNOBS; results are wrong for knobs != 0):
#   KNOBS="0 16 80" TAG=x bash tools/gpu_trace_knobs.sh
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-tk}
: > $O/${T}_trace.txt
for kn in ${KNOBS:-0}; do
  CPDGPU_F32F_KNOBS=$kn CPDGPU_SEED_TRACE=1 timeout 300 python bench.py --config ${CONFIG:-c5} --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 2>&1 \
    | grep "trace\]" | tail -1 | sed "s/^/knobs=$kn /" >> $O/${T}_trace.txt
done
