# dev: GEMM micro-bench (v1 vs v2) + scale probe
python -c "import __graft_entry__ as g; g.build()" || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2509_11152_b200/csrc -I include scripts/kbench.cu -L paper_2509_11152_b200 -lh2f -Xlinker -rpath=$PWD/paper_2509_11152_b200 -o /tmp/kbench || exit 1
echo "== v1"; H2F_GEMM_V1=1 /tmp/kbench
echo "== v2"; /tmp/kbench
timeout ${PROBE_TIMEOUT:-1500} python scripts/scale_probe.py ${PROBE:-helmholtz3d:32768:kappa=0.0} > gpurun_out/scale.log 2> gpurun_out/scale.err
echo "exit $?"
grep case gpurun_out/scale.log | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    print(d['case'], 'fact', d['fact_s'], 'solve', d['solve_s'], 'e_b', d['e_b'], 'raw', d['e_b_raw'], 'top', d['top'], 'batches', d['batches'])
    print('  ', {k: v[0] for k, v in list(d['kernels'].items())[:14]})
    print('  ', {k: v[0] for k, v in list(d['solve_kernels'].items())[:14]})
"
