mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
H2F_LEVEL_PROF=1 timeout 900 python scripts/scale_probe.py helmholtz3d:131072:kappa=0.0 > gpurun_out/scale.log 2> gpurun_out/scale.err
python -c "
import json; d=json.loads(open('gpurun_out/scale.log').readline()); print('fact', d['fact_s'], 'solve', d['solve_s'], 'e_b', d['e_b'], d['e_b_raw']); print({k: v[0] for k, v in list(d['kernels'].items())[:12]})"
