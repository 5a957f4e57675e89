"""Backward error of the GPU path vs the oracle across sizes (dev probe)."""
import sys, time, json
import numpy as np
sys.path.insert(0, '.')
import paper_2509_11152_b200 as H
from threadpoolctl import threadpool_limits

fam = sys.argv[1]
over = {}
ns = []
for a in sys.argv[2:]:
    if '=' in a:
        k, v = a.split('='); over[k] = float(v) if '.' in v else int(v)
    else:
        ns.append(int(a))
for n in ns:
    tree, part, spec, h2, prm = H.build_problem(fam, n, **over)
    x_ref = np.random.Generator(np.random.Philox(7)).standard_normal(n)
    b = H.matvec(h2, x_ref)
    t0 = time.perf_counter()
    fac = H.factorize(h2, prm["eps_lu"])
    tf = time.perf_counter() - t0
    x0 = H.solve(fac, b)
    x = H.refined_solve(h2, fac, b, steps=1)
    eb0 = np.linalg.norm(H.matvec(h2, x0) - b) / np.linalg.norm(b)
    eb = np.linalg.norm(H.matvec(h2, x) - b) / np.linalg.norm(b)
    out = {"n": n, "fam": fam, "over": over, "fact_s": round(tf, 3), "e_b_raw": eb0, "e_b": eb,
           "eps_fill": fac.eps_fill, "top": fac.top_size, "max_rank": [r.max_rank for r in fac.records],
           "batches": [r.nbatches for r in fac.records]}
    if n <= 8192:
        from oracle import h2_oracle as O
        with threadpool_limits(1):
            t0 = time.perf_counter()
            of = O.factorize(h2, prm["eps_lu"])
            ox0 = O.substitute(of, b)
            ox = O.refined_solve(h2, of, b, steps=1)
            out["oracle_s"] = round(time.perf_counter() - t0, 2)
        out["o_e_b_raw"] = np.linalg.norm(H.matvec(h2, ox0) - b) / np.linalg.norm(b)
        out["o_e_b"] = np.linalg.norm(H.matvec(h2, ox) - b) / np.linalg.norm(b)
        out["o_batches"] = [r.nbatches for r in of.records]
        out["o_max_rank"] = [r.max_rank for r in of.records]
        out["x_rel"] = float(np.linalg.norm(x - ox) / np.linalg.norm(ox))
    print(json.dumps(out), flush=True)
