# dev: ncu --set full of the first GEMM launch of the micro-bench, then the dense bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I paper_2509_11152_b200/csrc -I include scripts/kbench.cu -L paper_2509_11152_b200 -lh2f -Xlinker -rpath=$PWD/paper_2509_11152_b200 -o /tmp/kbench || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tasks_kernel -s 1 -c 1 -o gpurun_out/kbench_gemm -f /tmp/kbench > gpurun_out/ncu_kbench.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/ncu_kbench.log
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python scripts/dense_bench.py svd 2>&1 | tee gpurun_out/dense_bench.log
