# dev loop: build, smoke, gpu tests, scale probe (per-level profile on stderr)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
H2F_LEVEL_PROF=1 timeout ${PROBE_TIMEOUT:-1500} python scripts/scale_probe.py ${PROBE:-cov2d:16384 helmholtz3d:32768:kappa=0.0} > gpurun_out/scale.log 2> gpurun_out/scale.err
echo "exit $?" >> gpurun_out/scale.log
tail -3 gpurun_out/smoke.log; tail -15 gpurun_out/pytest_gpu.log; cut -c1-2500 gpurun_out/scale.log; grep level gpurun_out/scale.err | cut -c1-400
