#!/bin/bash
# GPU round trip used during development: parity suite + per-config bench lines.
cd "$(dirname "$0")/.."
python -m pytest tests -m gpu -q -x -k "not slow" 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
: > gpurun_out/bench.txt
for c in ${CONFIGS:-c2 c1 c3}; do
  python bench.py --config $c --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/bench.txt 2>&1
done
