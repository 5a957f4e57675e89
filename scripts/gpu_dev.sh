# dev loop: build, gpu tests, dense + gemm micro-benchmarks, optional probe
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python scripts/dense_bench.py ${DENSE:-svd qr cmp} 2>&1 | tee gpurun_out/dense_bench.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2509_11152_b200/csrc -I include scripts/kbench.cu -L paper_2509_11152_b200 -lh2f -Xlinker -rpath=$PWD/paper_2509_11152_b200 -o /tmp/kbench && /tmp/kbench
if [ -n "$PROBE" ]; then
  H2F_LEVEL_PROF=1 timeout ${PROBE_TIMEOUT:-1500} python scripts/scale_probe.py $PROBE > gpurun_out/scale.log 2> gpurun_out/scale.err
  echo "probe exit $?"; python scripts/summ.py gpurun_out/scale.log gpurun_out/scale.err
fi
