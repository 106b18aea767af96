#!/bin/bash
# the reference's own test sources and acceptance binary with mttkrp.cpp / als.cpp
# replaced by the drop-in over libcpdgpu.so (built here, oracle/_ref), then the GPU
# suite and the default bench line
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-dropin}
(cd oracle/_ref && timeout 600 ./cpd_tests_gpu > ../../$O/${T}_cpd_tests_gpu.txt 2>&1; echo "rc=$?" >> ../../$O/${T}_cpd_tests_gpu.txt)
(cd oracle/_ref && timeout 600 ./cpd_acceptance_gpu > ../../$O/${T}_cpd_acceptance_gpu.txt 2>&1; echo "rc=$?" >> ../../$O/${T}_cpd_acceptance_gpu.txt)
if [ "${TESTS:-1}" = 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/${T}_pytest_gpu.txt 2>&1
  echo "rc=$?" >> $O/${T}_pytest_gpu.txt
fi
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/${T}_bench_c5.json 2> $O/${T}_bench_c5.err
