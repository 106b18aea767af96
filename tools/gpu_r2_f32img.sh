#!/bin/bash
# tiled operand image: fp32 parity (+ c5 full size), watchdog tests, c5 bench, stream-floor knob
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-img}
timeout 900 python -m pytest tests/test_gpu_f32.py tests/test_gpu_watchdog.py tests/test_gpu_i8.py -q -x -s -p no:cacheprovider > $O/${T}_pytest.txt 2>&1
echo "rc=$?" >> $O/${T}_pytest.txt
KNOBS="0 32 16" TAG=${T}_knobs bash tools/gpu_knobs.sh
