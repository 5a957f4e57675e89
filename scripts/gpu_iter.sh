timeout 1200 python -m pytest tests/test_gpu_dense.py tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q > gpurun_out/it_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it_pytest.log
for i in 1 2; do timeout 800 python scripts/level_profile.py 2>&1 | grep -E "factorize|gemm_schur |gemm_project|gemm_top" ; done > gpurun_out/it_lp.log
