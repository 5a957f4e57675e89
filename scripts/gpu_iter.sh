python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/smoke.log; tail -15 gpurun_out/pytest_gpu.log
timeout 1200 python scripts/scale_probe.py ${PROBE:-cov2d:16384 helmholtz3d:8192:kappa=0.0 helmholtz3d:32768:kappa=0.0} > gpurun_out/scale.log 2>&1
echo "exit $?" >> gpurun_out/scale.log
cat gpurun_out/scale.log
