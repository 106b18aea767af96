#!/bin/bash
# One GPU round trip: adapter suite, full bench lines (c2 default with e2e + CPU
# baseline; c4 ALS), then — each only after its command exited 0 — the ncu launch
# list of the c2 bench and one `--set full` capture of the seed kernel.
cd "$(dirname "$0")/.."
O=gpurun_out
mkdir -p $O
python -m pytest tests/test_cpp_adapter.py -m gpu -q -x 2>&1 | tail -5 > $O/pytest_cpp.txt
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --config c4 --steps 20 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
for c in ${PROFILE_CONFIGS:-c2}; do
  if python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/pre_$c.json 2>&1; then
    ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$c.csv \
      python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch_$c.log 2>&1
    ncu --set full --clock-control none --import-source on -k regex:seed_f64 -s 6 -c 1 -o $O/seed_$c -f \
      python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_full_$c.log 2>&1
  fi
done
