# re-entry check at HEAD: smoke, gpu tests, config-2 bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_recheck.log 2> gpurun_out/bench_recheck.err; echo "bench exit $?"
cut -c1-900 gpurun_out/bench_recheck.log
