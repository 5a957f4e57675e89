# compute-sanitizer memcheck + racecheck of the smoke invocation (cov2d n=1024)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 compute-sanitizer --tool memcheck --print-limit 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck_smoke.log 2>&1; echo "memcheck exit $?" >> gpurun_out/memcheck_smoke.log
tail -4 gpurun_out/memcheck_smoke.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/racecheck_smoke.log 2>&1; echo "racecheck exit $?" >> gpurun_out/racecheck_smoke.log
tail -4 gpurun_out/racecheck_smoke.log
timeout 600 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_gpu.log
