# round-end evidence at HEAD: full GPU tests, smoke, config-2 bench (N=1)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/ev_bench_c2.json 2> gpurun_out/ev_bench_c2.err
