#!/bin/bash
# int8 fused seed: parity suite + c1-c3 timings (int8 vs CPDGPU_NO_I8=1 DMMA)
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "not slow" 2>&1 | tail -15 > $O/pytest_i8.txt
: > $O/bench_i8.txt
for c in ${CONFIGS:-c2 c1 c3}; do
  CPDGPU_I8=1 timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> $O/bench_i8.txt 2>> $O/bench_i8.err
  CPDGPU_I8=0 timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-alg1 >> $O/bench_i8.txt 2>> $O/bench_i8.err
done
