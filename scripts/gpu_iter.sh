timeout 1500 python -m pytest tests/test_gpu_dense.py tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q > gpurun_out/it_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it_pytest.log
timeout 800 python scripts/level_profile.py 2>&1 | grep -oE "factorize \(profiler off\).*|jacobi_svd_coop +[0-9.]+|qr_r_blocked +[0-9.]+" | tr '\n' ' ' > gpurun_out/it_lp.log
