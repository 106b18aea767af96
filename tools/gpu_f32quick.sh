#!/bin/bash
# fp32 path parity (all f32 GPU tests incl. c5 full size) + the c5 bench line + launch list
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-f32q}
timeout 900 python -m pytest tests/test_gpu_f32.py tests/test_gpu_sharded.py tests/test_gpu_sharded_abi.py -q -x -s -p no:cacheprovider > $O/${T}_pytest.txt 2>&1
echo "rc=$?" >> $O/${T}_pytest.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-alg1 > $O/${T}_bench.json 2> $O/${T}_bench.err
B="python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1"
if timeout 300 $B > /dev/null 2>&1; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file $O/${T}_launches.csv $B > /dev/null 2>&1
fi
