#!/bin/bash
# Round-2 measurement set on one B200 (each ncu pass only after its command exited 0):
# GPU suite + smoke, the driver's default bench (c5) and its reference arm, the other
# configs, the N=2 path functionally on the one GPU (BENCH_FUNCTIONAL_1GPU: gloo
# host all-reduce through the library communicator), launch lists, ncu captures.
cd "$(dirname "$0")/.."
O=gpurun_out; T=${TAG:-r02b}
mkdir -p $O
nvidia-smi > $O/${T}_smi.txt 2>&1
if [ "${TESTS:-1}" = 1 ]; then
  timeout 1500 python -m pytest ${TESTFILES:-tests} -m gpu -q -p no:cacheprovider > $O/${T}_pytest_gpu.txt 2>&1
  echo "rc=$?" >> $O/${T}_pytest_gpu.txt
  timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.txt 2>&1
  echo "rc=$?" >> $O/${T}_smoke.txt
fi
if [ "${BENCH:-1}" = 1 ]; then
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/${T}_bench_c5.json 2> $O/${T}_bench_c5.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/${T}_ref_c5.json 2> $O/${T}_ref_c5.err
fi
for c in ${CONFIGS-c1 c2 c3 c4}; do
  timeout 900 python bench.py --config $c --steps 50 --warmup 5 > $O/${T}_bench_$c.json 2> $O/${T}_bench_$c.err
done
[ "${BENCH:-1}" = 1 ] && timeout 600 python bench.py --impl reference --config c2 --steps 5 --warmup 1 > $O/${T}_ref_c2.json 2> $O/${T}_ref_c2.err
for c in ${N2CONFIGS-c5 c2 c4}; do
  BENCH_FUNCTIONAL_1GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --config $c --steps 3 --warmup 3 --no-e2e \
    --no-cpu-baseline --no-alg1 > $O/${T}_n2functional_$c.json 2> $O/${T}_n2functional_$c.err
done
for c in ${LAUNCHCONFIGS-c5 c2 c3}; do
  B="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1"
  if timeout 300 $B > /dev/null 2>&1; then
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/${T}_launches_$c.csv \
      $B > /dev/null 2>&1
  fi
done
B="python bench.py --config c2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1"
if [ "${NCU:-1}" = 1 ] && timeout 300 $B > /dev/null 2>&1; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"seed_i8" -s 2 -c 1 -o $O/${T}_seed_c2 -f \
    $B > $O/${T}_ncu_seed_c2.log 2>&1
fi
B="python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1"
if [ "${NCU5:-1}" = 1 ] && timeout 300 $B > /dev/null 2>&1; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"seed_f32i" -s 2 -c 1 -o $O/${T}_seed_c5 -f \
    $B > $O/${T}_ncu_seed_c5.log 2>&1
fi
echo done > $O/${T}_done.txt
