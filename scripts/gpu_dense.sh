# dev: dense kernel micro-bench, ncu of the block Jacobi + hh panel, e_b variants with pivot ratios
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python scripts/dense_bench.py svd qr cmp 2>&1 | tee gpurun_out/dense_bench.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi_block -s 2 -c 1 -o gpurun_out/jacobi_block -f python scripts/dense_bench.py svd > gpurun_out/ncu_jac.log 2>&1; echo "ncu jac exit $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hh_panel -s 40 -c 2 -o gpurun_out/hh_panel -f python scripts/dense_bench.py cmp > gpurun_out/ncu_hh.log 2>&1; echo "ncu hh exit $?"
timeout 1500 python scripts/variants_probe.py helmholtz3d 131072 kappa=0.0 ${VARS:-"V:H2F_LU_BLOCKED_MIN=100000,H2F_TRSM_DMMA_MIN=100000"} > gpurun_out/var.log 2> gpurun_out/var.err
echo "var exit $?"; cat gpurun_out/var.log; tail -3 gpurun_out/var.err
