mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
echo "== JB default"; timeout 600 python scripts/dense_bench.py svd 2>&1 | grep "path=1"
echo "== JB4 everywhere"; H2F_JACOBI_JB4_MIN_N=0 timeout 600 python scripts/dense_bench.py svd 2>&1 | grep "path=1"
H2F_JACOBI_JB4_MIN_N=300 H2F_LEVEL_PROF=1 timeout 900 python scripts/scale_probe.py helmholtz3d:131072:kappa=0.0 > gpurun_out/scale.log 2> gpurun_out/scale.err
echo "probe exit $?"; grep -o "jacobi_svd_coop=[0-9.]*" gpurun_out/scale.err | tr '\n' ' '
python -c "
import json; d=json.loads(open('gpurun_out/scale.log').readline()); print('fact', d['fact_s'], 'e_b', d['e_b'], d['e_b_raw'])"
