# Jacobi 4-row-block threshold sweep on config 2 (factorization wall time)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for t in 512 320 1024; do
  H2F_JACOBI_JB4_MIN_N=$t timeout 600 python scripts/scale_probe.py helmholtz3d:131072:kappa=0.0 > gpurun_out/jb4_$t.log 2> gpurun_out/jb4_$t.err
  python -c "
import json; d=json.loads(open('gpurun_out/jb4_$t.log').readline()); print('jb4_min_n=$t fact', d['fact_s'], 'e_b', d['e_b'], d['e_b_raw'])" | tee -a gpurun_out/jb4_sweep.txt
done
