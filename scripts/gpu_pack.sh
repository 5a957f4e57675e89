mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I paper_2509_11152_b200/csrc -I include scripts/kbench.cu -L paper_2509_11152_b200 -lh2f -Xlinker -rpath=$PWD/paper_2509_11152_b200 -o /tmp/kbench
/tmp/kbench
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
rm -f gpurun_out/prof_c2.log
H2F_PROF_LOG=gpurun_out/prof_c2.log timeout 900 python scripts/scale_probe.py helmholtz3d:131072:kappa=0.0 > gpurun_out/scale.log 2> gpurun_out/scale.err
echo "probe exit $?"; python scripts/prof_log_summary.py gpurun_out/prof_c2.log gemm_schur
python -c "
import json; d=json.loads(open('gpurun_out/scale.log').readline()); print('fact', d['fact_s'], 'solve', d['solve_s'], 'e_b', d['e_b'], d['e_b_raw'])"
timeout 600 python scripts/multi_rhs_probe.py 256
