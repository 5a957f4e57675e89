"""Spread of the backward error over rounding-level draws of the same
operator (dev probe): the dense near field is multiplied elementwise by
(1 + p z), z ~ N(0,1) symmetrised on diagonal blocks, p = 1e-14; each draw is
factored and solved on the GPU.  Same perturbation as scripts/oracle_big.py
perturb=... for the CPU oracle."""
import copy, gc, json, sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_2509_11152_b200 as H

fam, n, ndraws = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
over = {}
SAVE = set()
FIRST = 0
for a in sys.argv[4:]:
    k, v = a.split('=')
    if k == "first":
        FIRST = int(v)
        continue
    if k == "save":
        SAVE = {int(t) for t in v.split(',')}
        continue
    over[k] = float(v) if '.' in v or 'e' in v else int(v)
tree, part, spec, h2, prm = H.build_problem(fam, n, **over)
x_ref = np.random.Generator(np.random.Philox(7)).standard_normal(n)
for d in range(FIRST, ndraws):
    h2p = copy.copy(h2)
    object.__setattr__(h2p, "_h2f_device", None)
    if d > 0:
        rng = np.random.default_rng(d)
        dense = {}
        for key in sorted(h2.dense):
            blk = h2.dense[key]
            z = rng.standard_normal(blk.shape)
            if key[0] == key[1]:
                z = 0.5 * (z + z.T)
            dense[key] = blk * (1.0 + 1e-14 * z)
        h2p.dense = dense
    b = H.matvec(h2p, x_ref)
    t0 = time.perf_counter()
    fac = H.factorize(h2p, prm["eps_lu"])
    tf = time.perf_counter() - t0
    x0 = H.solve(fac, b)
    x = H.refined_solve(h2p, fac, b, steps=1)
    eb0 = float(np.linalg.norm(H.matvec(h2p, x0) - b) / np.linalg.norm(b))
    eb = float(np.linalg.norm(H.matvec(h2p, x) - b) / np.linalg.norm(b))
    print(json.dumps({"draw": d, "perturb": 0.0 if d == 0 else 1e-14, "fact_s": round(tf, 2), "e_b_raw": eb0,
                      "e_b": eb, "levels": [[r.level, r.nbatches, r.max_rank] for r in fac.records]}), flush=True)
    if d in SAVE:
        save = {"x": x, "x0": x0}
        for rec in fac.records:
            cl = list(rec.clusters)
            save[f"L{rec.level}_clusters"] = np.array(cl)
            save[f"L{rec.level}_size"] = np.array([rec.size[c] for c in cl])
            save[f"L{rec.level}_r"] = np.array([rec.factors[c].r for c in cl])
            save[f"L{rec.level}_batches"] = np.concatenate([np.array(bb) for bb in rec.batches])
            save[f"L{rec.level}_blen"] = np.array([len(bb) for bb in rec.batches])
        np.savez(f"gpurun_out/draw{d}_structure.npz", **save)
    del fac, h2p
    gc.collect()
