# quick fp64 check: gradient parity suites, c1-c3 seed timings, c2 per-warp trace
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_gradient.py tests/test_gpu_random_shapes.py tests/test_gpu_sharded.py -x -q -m gpu 2>&1 | tail -2
for c in c2 c1 c3; do
  python bench.py --config $c --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print(d['config']['workload'], round(d['ms_per_step']*1e3,1), 'us/step  seed', round(r['kernel_ms']*1e3,1), 'us', r['bound'], round(r['frac'],3))"
done
python tools/seed_trace.py c2 2>&1 | tail -2; CPDGPU_PDL=0 python tools/seed_trace.py c2 2>&1 | tail -1
python tools/timeline.py c2 6 2>&1 | tail -3
