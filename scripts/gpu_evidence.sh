# round-end evidence at HEAD: full GPU tests, config-2 bench (N=1), configs 1 and 5
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev_pytest_gpu.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/ev_bench_c2.json 2> gpurun_out/ev_bench_c2.err
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 > gpurun_out/ev_bench_c1.json 2> gpurun_out/ev_bench_c1.err
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu > gpurun_out/ev_bench_c5.json 2> gpurun_out/ev_bench_c5.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1
