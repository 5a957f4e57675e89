# full GPU test suite, then the config-2 bench line (N=1)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/rc_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc_pytest_gpu.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/rc_bench_c2.json 2> gpurun_out/rc_bench_c2.err; echo "bench rc=$?" >> gpurun_out/rc_bench_c2.err
