# config-2 evidence: kernel micro-bench, launch list of one step, ncu full of the Schur GEMM
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I paper_2509_11152_b200/csrc -I include scripts/kbench.cu -L paper_2509_11152_b200 -lh2f -Xlinker -rpath=$PWD/paper_2509_11152_b200 -o /tmp/kbench && /tmp/kbench | tee gpurun_out/kbench.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python scripts/one_step.py 2 > gpurun_out/ncu_launch_c2.log 2>&1
echo "ncu launches exit $?"
python scripts/launch_summary.py gpurun_out/launches_c2.csv "one step of config 2" | head -30
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_tasks_kernel -s 2600 -c 6 \
    -o gpurun_out/prof_gemm_c2 -f python scripts/one_step.py 2 > gpurun_out/ncu_gemm_c2.log 2>&1
echo "ncu gemm exit $?"
python scripts/ncu_summary.py gpurun_out/prof_gemm_c2.ncu-rep
