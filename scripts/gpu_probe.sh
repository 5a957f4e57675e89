python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python scripts/scale_probe.py ${PROBE} > gpurun_out/scale.log 2>&1
echo "exit $?" >> gpurun_out/scale.log
cat gpurun_out/scale.log
