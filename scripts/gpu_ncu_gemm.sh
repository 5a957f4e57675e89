python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I paper_2509_11152_b200/csrc -I include scripts/kbench.cu -L paper_2509_11152_b200 -lh2f -Xlinker -rpath=$PWD/paper_2509_11152_b200 -o /tmp/kbench || exit 1
/tmp/kbench
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tasks_kernel -s 1 -c 1 -o gpurun_out/kbench_leaf -f /tmp/kbench schur_leaf > gpurun_out/ncu_kbench.log 2>&1; echo "ncu exit $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi_block -c 1 -o gpurun_out/jacobi_block -f python scripts/dense_bench.py svd > gpurun_out/ncu_jac.log 2>&1; echo "ncu jac exit $?"
timeout 600 python scripts/dense_bench.py qr cmp 2>&1 | tee gpurun_out/dense_bench.log
