# round-1 checkpoint: build, smoke, gpu tests, config-2 bench + reference arm
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep "Model name"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/smoke.log; tail -30 gpurun_out/pytest_gpu.log
timeout 1800 python bench.py --config ${CFG:-2} --steps 3 --warmup 3 > gpurun_out/bench.log 2> gpurun_out/bench.err
echo "exit $?" >> gpurun_out/bench.log
cat gpurun_out/bench.log; tail -20 gpurun_out/bench.err
