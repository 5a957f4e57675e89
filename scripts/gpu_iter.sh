# development iteration: parity + sharded tests, then the per-level profile of config 2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q > gpurun_out/it_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it_pytest.log
timeout 800 python scripts/level_profile.py > gpurun_out/it_lp.log 2>&1
