# round-end evidence at HEAD: full GPU tests, config-2 bench (N=1), config 1 bench, launch list of one config-2 step
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev_pytest_gpu.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/ev_bench_c2.json 2> gpurun_out/ev_bench_c2.err
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 > gpurun_out/ev_bench_c1.json 2> gpurun_out/ev_bench_c1.err
