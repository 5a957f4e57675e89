python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python scripts/scale_probe.py cov2d:16384 cov3d:8192 helmholtz3d:8192:kappa=0.0 cov2d:65536 helmholtz3d:32768:kappa=0.0 > gpurun_out/scale.log 2>&1
echo "exit $?" >> gpurun_out/scale.log
cat gpurun_out/scale.log
