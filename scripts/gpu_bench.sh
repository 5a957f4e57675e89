python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py --config ${CFG:-1} --steps 3 --warmup 3 > gpurun_out/bench.log 2> gpurun_out/bench.err
echo "exit $?" >> gpurun_out/bench.log
timeout 300 python bench.py --config ${CFG:-1} --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1
cat gpurun_out/bench.log gpurun_out/bench_ref.log; tail -5 gpurun_out/bench.err
