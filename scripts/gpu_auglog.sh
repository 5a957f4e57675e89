# dev: per-cluster augmentation shapes + per-level kernel profile at a given size
python -c "import __graft_entry__ as g; g.build()" || exit 1
rm -f gpurun_out/aug_*.log
for c in ${PROBE:-helmholtz3d:131072:kappa=0.0}; do
  H2F_AUG_LOG=gpurun_out/aug_$(echo $c | cut -d: -f1-2 | tr : _).log H2F_LEVEL_PROF=1 timeout 1500 python scripts/scale_probe.py $c > gpurun_out/auglog_scale.log 2> gpurun_out/auglog_scale.err
done
echo "exit $?" >> gpurun_out/auglog_scale.log
cut -c1-3000 gpurun_out/auglog_scale.log; grep level gpurun_out/auglog_scale.err | cut -c1-600; wc -l gpurun_out/aug_*.log
