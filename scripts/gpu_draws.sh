mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1800 python scripts/draws_probe.py helmholtz3d 131072 ${NDRAWS:-7} kappa=0.0 > gpurun_out/draws.log 2> gpurun_out/draws.err
echo "draws exit $?"; python - <<'PY'
import json
for l in open('gpurun_out/draws.log'):
    d=json.loads(l); print(d['draw'], d['fact_s'], 'e_b %.3g raw %.3g' % (d['e_b'], d['e_b_raw']), d['levels'][-1])
PY
tail -3 gpurun_out/draws.err
