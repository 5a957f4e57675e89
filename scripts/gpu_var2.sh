mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python scripts/variants_probe.py helmholtz3d 131072 kappa=0.0 "V:H2F_SVD_SMEM_MAX=96" "V:H2F_SVD_SMEM_MAX=64" "V:H2F_SVD_SMEM_MAX=32" > gpurun_out/var.log 2> gpurun_out/var.err
echo "var exit $?"; cut -c1-200 gpurun_out/var.log; python - <<'PY'
import json
for l in open('gpurun_out/var.log'):
    d=json.loads(l); print(d['variant'], d.get('fact_s'), d.get('e_b'), d.get('e_b_raw'))
PY
