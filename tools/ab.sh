# A/B seed timing on one box: tools/ab.sh "A B ..." "c2 c1" reps
cd $GRAFT_REPO_ROOT
for rep in $(seq ${3:-2}); do
  for c in $2; do
    for v in $1; do
      CPDGPU_LIB=tools/bisect_$v.so python bench.py --config $c --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-alg1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print('$v', d['config']['workload'], round(d['ms_per_step']*1e3,1), 'us  seed', round(r['kernel_ms']*1e3,1))"
    done
  done
done
