# round-1 closing evidence at HEAD: smoke, gpu tests, bench (config 2, reference arm, config 5),
# launch list of one config-2 step, backward-error draws (structure of draws 0 and 2 saved)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_final.log 2> gpurun_out/bench_final.err; echo "bench exit $?"
cut -c1-700 gpurun_out/bench_final.log
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_final.log 2>&1; echo "ref exit $?"
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/bench_c5_final.log 2> gpurun_out/bench_c5.err; echo "c5 exit $?"
cut -c1-300 gpurun_out/bench_c5_final.log
timeout 1500 python scripts/draws_probe.py helmholtz3d 131072 ${NDRAWS:-5} kappa=0.0 save=0,2 > gpurun_out/draws.log 2> gpurun_out/draws.err
echo "draws exit $?"; cut -c1-250 gpurun_out/draws.log
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_final.csv \
    python scripts/one_step.py 2 > gpurun_out/ncu_launch_final.log 2>&1
echo "ncu launches exit $?"
python scripts/launch_summary.py gpurun_out/launches_c2_final.csv "final" 2>/dev/null | head -12
