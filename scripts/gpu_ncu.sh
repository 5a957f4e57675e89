python -c "import __graft_entry__ as g; g.build()"
timeout 600 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench.log 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.log
# launch list of one bench step (cold cache, serialised): shares only
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --config 1 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_launch_run.log 2>&1
echo "ncu launches exit $?" >> gpurun_out/bench.log
# full capture of the top kernels (3 launches each)
for k in jacobi_smem_kernel qr_r_smem_kernel gemm_tasks_kernel; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 2 \
    -o gpurun_out/prof_$k python bench.py --config 1 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_$k.log 2>&1
echo "ncu $k exit $?" >> gpurun_out/bench.log
done
cat gpurun_out/bench.log
