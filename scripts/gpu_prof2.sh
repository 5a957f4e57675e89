python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2509_11152_b200/csrc -I include scripts/kbench.cu -L paper_2509_11152_b200 -lh2f -Xlinker -rpath=$PWD/paper_2509_11152_b200 -o /tmp/kbench && /tmp/kbench
timeout 600 python scripts/dense_bench.py ${DENSE:-svd cmp} 2>&1 | tee gpurun_out/dense_bench.log
rm -f gpurun_out/prof_*.log
for c in ${PROBE:-helmholtz3d:32768:kappa=0.0}; do
  H2F_PROF_LOG=gpurun_out/prof_$(echo $c | cut -d: -f1-2 | tr : _).log H2F_LEVEL_PROF=1 timeout 1500 python scripts/scale_probe.py $c > gpurun_out/scale.log 2> gpurun_out/scale.err
  python scripts/summ.py gpurun_out/scale.log gpurun_out/scale.err
done
