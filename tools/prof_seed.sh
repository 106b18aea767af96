cd $GRAFT_REPO_ROOT
O=gpurun_out
python bench.py --config c2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 > $O/p_c2.json 2>&1 || exit 1
python -c "import json; d=json.loads(open('$O/p_c2.json').readline()); print(d['ms_per_step'], d['roofline']['kernel_ms'])"
ncu --set full --import-source on --clock-control none -k regex:seed_f64 -s 6 -c 1 -o $O/pair_c2 -f python bench.py --config c2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 > /dev/null 2>&1
ls -la $O/pair_c2.ncu-rep
