"""Factor one large case under several kernel-path settings (dev probe):
prints e_b raw/refined and per-level structure; saves the default run's
structure + solution to gpurun_out/ for comparison with the oracle."""
import os, sys, time, json
import numpy as np
sys.path.insert(0, '.')
import paper_2509_11152_b200 as H

fam, n = sys.argv[1], int(sys.argv[2])
over, variants = {}, [""]
for a in sys.argv[3:]:
    if a.startswith("V:"):
        variants.append(a[2:])
    else:
        k, v = a.split('='); over[k] = float(v) if '.' in v else int(v)
tree, part, spec, h2, prm = H.build_problem(fam, n, **over)
x_ref = np.random.Generator(np.random.Philox(7)).standard_normal(n)
b = H.matvec(h2, x_ref)
base = dict(os.environ)
for vi, var in enumerate(variants):
    os.environ.clear(); os.environ.update(base)
    for kv in filter(None, var.split(',')):
        k, v = kv.split('='); os.environ[k] = v
    t0 = time.perf_counter()
    try:
        fac = H.factorize(h2, prm["eps_lu"])
    except Exception as e:
        print(json.dumps({"variant": var, "error": repr(e)}), flush=True); continue
    tf = time.perf_counter() - t0
    x0 = H.solve(fac, b)
    x = H.refined_solve(h2, fac, b, steps=1)
    eb0 = np.linalg.norm(H.matvec(h2, x0) - b) / np.linalg.norm(b)
    eb = np.linalg.norm(H.matvec(h2, x) - b) / np.linalg.norm(b)
    piv = []
    for rec in fac.records:
        worst = (np.inf, -1)
        for c, f in rec.factors.items():
            if f.r:
                lu = f.lu
                ratio = float(np.abs(np.diag(lu)).min() / max(np.abs(lu).max(), 1e-300))
                worst = min(worst, (ratio, c))
        piv.append([rec.level, worst[0], worst[1]])
    if fac.top_size:
        tl = fac.top_lu
        piv.append(["top", float(np.abs(np.diag(tl)).min() / np.abs(tl).max()), -1])
    print(json.dumps({"variant": var, "pivot_ratio_min": piv, "fact_s": round(tf, 2), "e_b_raw": eb0, "e_b": eb, "top": fac.top_size,
                      "levels": [[r.level, r.nbatches, r.max_rank] for r in fac.records]}), flush=True)
    if vi == 0:
        save = {"x": x, "x0": x0}
        for rec in fac.records:
            cl = list(rec.clusters)
            save[f"L{rec.level}_r"] = np.array([rec.factors[c].r for c in cl])
            save[f"L{rec.level}_clusters"] = np.array(cl)
            save[f"L{rec.level}_batches"] = np.concatenate([np.array(bb) for bb in rec.batches])
        np.savez(f"gpurun_out/gpu_{fam}_{n}.npz", **save)
    del fac
