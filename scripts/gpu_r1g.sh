# more backward-error draws at HEAD (draws 5..11) + per-level device/host profile of config 2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python scripts/draws_probe.py helmholtz3d 131072 12 kappa=0.0 first=5 > gpurun_out/draws2.log 2> gpurun_out/draws2.err
echo "draws exit $?"; cut -c1-200 gpurun_out/draws2.log
H2F_LEVEL_PROF=1 timeout 900 python scripts/scale_probe.py helmholtz3d:131072:kappa=0.0 > gpurun_out/scale.log 2> gpurun_out/scale.err
echo "scale exit $?"; grep level gpurun_out/scale.err | cut -c1-600
