mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python scripts/variants_probe.py helmholtz3d 131072 kappa=0.0 "V:H2F_LU_BLOCKED_MIN=100000,H2F_TRSM_DMMA_MIN=100000" "V:H2F_HH_MIN_S=100000" "V:H2F_JACOBI_PAIRWISE=1" > gpurun_out/var.log 2> gpurun_out/var.err
echo "exit $?" >> gpurun_out/var.log
cat gpurun_out/var.log; tail -5 gpurun_out/var.err
