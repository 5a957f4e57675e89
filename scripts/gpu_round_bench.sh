# round evidence: bench config 2 (with cpu_baseline), reference arm, config 5, GEMM ncu on the micro-bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench exit $?"
cat gpurun_out/bench.log; tail -3 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?"; cat gpurun_out/bench_ref.log
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/bench_c5.log 2> gpurun_out/bench_c5.err; echo "c5 exit $?"; cat gpurun_out/bench_c5.log; tail -3 gpurun_out/bench_c5.err
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I paper_2509_11152_b200/csrc -I include scripts/kbench.cu -L paper_2509_11152_b200 -lh2f -Xlinker -rpath=$PWD/paper_2509_11152_b200 -o /tmp/kbench
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tasks_kernel -s 1 -c 1 -o gpurun_out/kbench_r150 -f /tmp/kbench schur_r150 > gpurun_out/ncu_kbench.log 2>&1; echo "ncu exit $?"
