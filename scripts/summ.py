"""Summarise scale_probe output (dev aid): python scripts/summ.py gpurun_out/scale.log [gpurun_out/scale.err]"""
import json, re, sys
for l in open(sys.argv[1]):
    if not l.startswith('{'):
        continue
    d = json.loads(l)
    print(d['case'], 'fact', d['fact_s'], 'solve', d['solve_s'], 'e_b', d['e_b'], 'raw', d.get('e_b_raw'),
          'top', d['top'], 'batches', d['batches'])
    print('   fact:', {k: v[0] for k, v in list(d['kernels'].items())[:14]})
    print('   solve:', {k: v[0] for k, v in list(d['solve_kernels'].items())[:8]})
if len(sys.argv) > 2:
    keys = ['gemm_schur', 'jacobi_svd_coop', 'jacobi_svd', 'complement', 'qr_r_blocked', 'trsm_eliminator',
            'lu_redundant']
    for l in open(sys.argv[2]):
        if not l.startswith('[level'):
            continue
        d = dict(re.findall(r'(\w+)=([\d.]+)', l))
        print(l.split(']')[0] + ']', l.split('wall ')[1].split(' s')[0], {k: d.get(k) for k in keys})
