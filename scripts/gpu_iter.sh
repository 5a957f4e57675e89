timeout 900 python -m pytest tests/test_gpu_boundary.py -x -q > gpurun_out/it_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/it_pytest.log
timeout 1500 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err
