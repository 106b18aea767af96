#!/bin/bash
# launch list (per-kernel device time, ncu --metrics gpu__time_duration.sum) of a short
# bench run per config, each only after the same command exited 0 without ncu
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-r02}
for c in ${CONFIGS:-c5}; do
  B="python bench.py --config $c --steps ${STEPS:-2} --warmup 3 --no-e2e --no-cpu-baseline --no-alg1"
  if $B > $O/${T}_pre_$c.json 2> $O/${T}_pre_$c.err; then
    ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-400} --csv --log-file $O/${T}_launches_$c.csv \
      $B > $O/${T}_ncu_launch_$c.log 2>&1
  fi
done
