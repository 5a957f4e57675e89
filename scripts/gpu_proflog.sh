mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
rm -f gpurun_out/prof_c2.log
H2F_PROF_LOG=gpurun_out/prof_c2.log timeout 900 python scripts/scale_probe.py helmholtz3d:131072:kappa=0.0 > gpurun_out/scale.log 2> gpurun_out/scale.err
echo "probe exit $?"
for k in gemm_schur gemm_project jacobi_svd_coop qr_r_blocked complement; do python scripts/prof_log_summary.py gpurun_out/prof_c2.log $k; done
