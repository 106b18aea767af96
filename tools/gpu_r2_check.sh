cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r2_pytest_gpu.txt
make -s -C tests/cpp && tests/cpp/_build/test_adapter > gpurun_out/r2_adapter.txt 2>&1
python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/r2_bench_c5.txt 2>&1
nvidia-smi -q -d CLOCK,POWER | head -60 > gpurun_out/r2_smi.txt
