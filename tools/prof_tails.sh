cd $GRAFT_REPO_ROOT
O=gpurun_out
python bench.py --config c2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:"prologue|tail_step" -s 9 -c 3 -o $O/tails_c2 -f python bench.py --config c2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_c2_now.csv python bench.py --config c2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-alg1 > /dev/null 2>&1
ls $O/tails_c2.ncu-rep
