# dev loop: gpu tests, GEMM micro-bench, config-2 bench, e_b variants with pivot ratios
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I paper_2509_11152_b200/csrc -I include scripts/kbench.cu -L paper_2509_11152_b200 -lh2f -Xlinker -rpath=$PWD/paper_2509_11152_b200 -o /tmp/kbench && /tmp/kbench | tee gpurun_out/kbench.log
timeout 1200 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench.log 2> gpurun_out/bench.err
echo "bench exit $?"; python -c "
import json; d=json.loads(open('gpurun_out/bench.log').readline()); print(d['value'], d['e2e'], d['roofline'], d['backward_error']); print({k:round(v['ms']) for k,v in d['kernels'].items()})"
timeout 1500 python scripts/variants_probe.py helmholtz3d 131072 kappa=0.0 ${VARS:-"V:H2F_LU_BLOCKED_MIN=100000,H2F_TRSM_DMMA_MIN=100000"} > gpurun_out/var.log 2> gpurun_out/var.err
echo "var exit $?"; cat gpurun_out/var.log; tail -3 gpurun_out/var.err
