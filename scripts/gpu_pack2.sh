mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I paper_2509_11152_b200/csrc -I include scripts/kbench.cu -L paper_2509_11152_b200 -lh2f -Xlinker -rpath=$PWD/paper_2509_11152_b200 -o /tmp/kbench
echo "== pack"; /tmp/kbench | head -4
echo "== nopack"; H2F_GEMM_NOPACK=1 /tmp/kbench | head -4
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
H2F_GEMM_NOPACK=1 timeout 900 python scripts/scale_probe.py helmholtz3d:131072:kappa=0.0 > gpurun_out/scale_np.log 2> gpurun_out/scale_np.err
python -c "
import json; d=json.loads(open('gpurun_out/scale_np.log').readline()); print('NOPACK fact', d['fact_s'], 'e_b', d['e_b'], d['e_b_raw'], d['kernels'].get('gemm_schur'))"
timeout 900 python scripts/scale_probe.py helmholtz3d:131072:kappa=0.0 > gpurun_out/scale.log 2> gpurun_out/scale.err
python -c "
import json; d=json.loads(open('gpurun_out/scale.log').readline()); print('PACK fact', d['fact_s'], 'e_b', d['e_b'], d['e_b_raw'], d['kernels'].get('gemm_schur'))"
timeout 600 python scripts/multi_rhs_probe.py 256
