#!/bin/bash
# fused fp32 seed: parity (small + c5 full size vs the streaming oracle), c5 timing,
# ablation knobs, ncu capture of the fused kernel
cd "$(dirname "$0")/.."
TAG=${TAG:-f32f}
timeout 300 python -m pytest tests/test_gpu_f32.py -q -x -k "not full_c5" > gpurun_out/${TAG}_pytest.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_pytest.txt
timeout 300 python -m pytest tests/test_gpu_f32.py -q -x -k "full_c5" > gpurun_out/${TAG}_c5.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_c5.txt
B="python bench.py --config c5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1"
: > gpurun_out/${TAG}_bench.txt
for k in ${KNOBS:-0 1 2 6 8 15}; do
  echo "knobs=$k" >> gpurun_out/${TAG}_bench.txt
  CPDGPU_F32F_KNOBS=$k timeout 300 $B >> gpurun_out/${TAG}_bench.txt 2>&1
done
if [ "${NCU:-1}" = 1 ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-seed_f32} -c 1 -o gpurun_out/${TAG}_c5 -f \
  python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-alg1 > gpurun_out/${TAG}_ncu.log 2>&1
fi
