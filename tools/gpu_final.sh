#!/bin/bash
# Round-end measurement set: full bench lines per config, launch list and ncu
# captures of the dominant kernels (each ncu only after its command exited 0).
cd "$(dirname "$0")/.."
O=gpurun_out
mkdir -p $O
python bench.py > $O/final_c2.json 2> $O/final_c2.err
python bench.py --config c1 --steps 100 --warmup 10 > $O/final_c1.json 2>/dev/null
python bench.py --config c3 --steps 50 --warmup 5 > $O/final_c3.json 2>/dev/null
python bench.py --config c4 --steps 20 --warmup 3 > $O/final_c4.json 2>/dev/null
python bench.py --config c5 --steps 10 --warmup 3 > $O/final_c5.json 2>/dev/null
python bench.py --impl reference --steps 5 --warmup 1 > $O/final_ref_c2.json 2>/dev/null
if python bench.py --config c2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 > $O/pre.json 2>&1; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/final_launches_c2.csv \
    python bench.py --config c2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 > /dev/null 2>&1
  ncu --set full --import-source on --clock-control none -k regex:"seed_i8|seed_f64" -s 6 -c 1 -o $O/final_seed_c2 -f \
    python bench.py --config c2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 > /dev/null 2>&1
fi
if python bench.py --config c5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 > $O/pre5.json 2>&1; then
  ncu --set full --import-source on --clock-control none -k regex:seed_f32 -s 2 -c 2 -o $O/final_seed_c5 -f \
    python bench.py --config c5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 > /dev/null 2>&1
fi
if python bench.py --config c4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/pre4.json 2>&1; then
  ncu --set full --import-source on --clock-control none -k regex:"seed_left_cols|seed_f64" -s 4 -c 2 -o $O/final_seed_c4 -f \
    python bench.py --config c4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
fi
# the fp64 DMMA pass on the configs where the int8 pass is the default (comparison lines)
for c in c2 c3; do
  CPDGPU_I8=0 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline > $O/final_dmma_$c.json 2>/dev/null
done
if CPDGPU_I8=0 python bench.py --config c2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 > $O/pre_dmma.json 2>&1; then
  CPDGPU_I8=0 ncu --set full --import-source on --clock-control none -k regex:seed_f64 -s 2 -c 1 -o $O/final_dmma_c2 -f \
    python bench.py --config c2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 > /dev/null 2>&1
fi
if python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 > $O/pre3.json 2>&1; then
  ncu --set full --import-source on --clock-control none -k regex:"seed_i8|seed_f64" -s 2 -c 1 -o $O/final_seed_c3 -f \
    python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 > /dev/null 2>&1
fi
