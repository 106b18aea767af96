#!/bin/bash
# Round-2 measurement set on one B200: GPU tests, the driver's default bench
# command (c5), launch list, and one ncu --set full capture of the c5 seed.
# Each ncu pass runs only after the same command exited 0 without ncu.
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-r02}
mkdir -p $O
nvidia-smi > $O/${T}_smi.txt 2>&1
if [ "${TESTS:-1}" = 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/${T}_pytest_gpu.txt 2>&1
  echo "rc=$?" >> $O/${T}_pytest_gpu.txt
  timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.txt 2>&1
  echo "rc=$?" >> $O/${T}_smoke.txt
fi
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/${T}_bench_c5.json 2> $O/${T}_bench_c5.err
echo "rc=$?" >> $O/${T}_bench_c5.err
for c in ${CONFIGS:-}; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 > $O/${T}_bench_$c.json 2> $O/${T}_bench_$c.err
done
B="python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1"
if timeout 300 $B > $O/${T}_pre_c5.json 2> $O/${T}_pre_c5.err; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${T}_launches_c5.csv \
    $B > $O/${T}_ncu_launch_c5.log 2>&1
  if [ "${NCU:-1}" = 1 ]; then
    timeout 900 ncu --set full --import-source on --clock-control none -k regex:seed_f32 -s 1 -c 1 -o $O/${T}_seed_c5 -f \
      $B > $O/${T}_ncu_seed_c5.log 2>&1
  fi
fi
echo done > $O/${T}_done.txt
