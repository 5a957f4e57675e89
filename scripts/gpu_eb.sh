mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python scripts/eb_probe.py helmholtz3d kappa=0.0 4096 8192 16384 32768 65536 131072 > gpurun_out/eb.log 2> gpurun_out/eb.err
echo "exit $?" >> gpurun_out/eb.log
cat gpurun_out/eb.log; tail -5 gpurun_out/eb.err
