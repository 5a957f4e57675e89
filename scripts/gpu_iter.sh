timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "matvec or norm or deterministic or solution" > gpurun_out/it_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it_pytest.log
timeout 800 python scripts/level_profile.py 2>&1 | grep -oE "factorize \(profiler off\).*|matvec_gemv=[0-9.]+" | tr '\n' ' ' > gpurun_out/it_mv.log
