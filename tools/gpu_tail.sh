#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-tail}
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/${T}_pytest.txt 2>&1
echo "rc=$?" >> $O/${T}_pytest.txt
for c in c5 c1 c4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-alg1 > $O/${T}_bench_$c.json 2>&1
done
B="python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1"
if timeout 300 $B > /dev/null 2>&1; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/${T}_launches_c5.csv $B > /dev/null 2>&1
fi
