"""Run the CPU oracle on a large case and save the structure + solution
(dev diagnostic; output outside the repo)."""
import sys, time, json, hashlib
import numpy as np
sys.path.insert(0, '/root/repo')
from threadpoolctl import threadpool_limits
import paper_2509_11152_b200.problem as P
from oracle import h2_oracle as O

fam, n, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
over = {}
perturb = 0.0
pseed = 1
decisions = None
for a in sys.argv[4:]:
    k, v = a.split('=')
    if k == "decisions":
        decisions = v
        O.DECISIONS = {}
        continue
    if k == "perturb":
        perturb = float(v)
        continue
    if k == "seed":
        pseed = int(v)
        continue
    over[k] = float(v) if '.' in v or 'e' in v else int(v)
t0 = time.perf_counter()
tree, part, spec, h2, prm = P.build_problem(fam, n, **over)
print("build", time.perf_counter() - t0, flush=True)
if perturb:
    # rounding-level perturbation of the dense near field (a different draw of
    # the same algorithm on an operator equal to working precision)
    rng = np.random.default_rng(pseed)
    for key in sorted(h2.dense):
        blk = h2.dense[key]
        z = rng.standard_normal(blk.shape)
        if key[0] == key[1]:
            z = 0.5 * (z + z.T)  # diagonal blocks stay symmetric
        h2.dense[key] = blk * (1.0 + perturb * z)
    print("perturbed dense blocks by", perturb, flush=True)
x_ref = np.random.Generator(np.random.Philox(7)).standard_normal(n)
with threadpool_limits(1):
    b = O.matvec(h2, x_ref)
    t0 = time.perf_counter()
    fac = O.factorize(h2, prm["eps_lu"])
    tf = time.perf_counter() - t0
    print("factor", tf, flush=True)
    x0 = O.substitute(fac, b)
    x = O.refined_solve(h2, fac, b, steps=1)
    eb0 = np.linalg.norm(O.matvec(h2, x0) - b) / np.linalg.norm(b)
    eb = np.linalg.norm(O.matvec(h2, x) - b) / np.linalg.norm(b)
save = {"x": x, "x0": x0, "b": b}
summary = {"n": n, "fam": fam, "over": over, "fact_s": tf, "e_b_raw": eb0, "e_b": eb, "eps_fill": fac.eps_fill,
           "norm": fac.norm_estimate, "top": fac.top_size, "digest": hashlib.sha256(x.tobytes()).hexdigest(),
           "levels": []}
for rec in fac.records:
    cl = list(rec.clusters)
    save[f"L{rec.level}_clusters"] = np.array(cl)
    save[f"L{rec.level}_size"] = np.array([rec.size[c] for c in cl])
    save[f"L{rec.level}_r"] = np.array([rec.factors[c].r for c in cl])
    save[f"L{rec.level}_batches"] = np.concatenate([np.array(bb) for bb in rec.batches])
    save[f"L{rec.level}_blen"] = np.array([len(bb) for bb in rec.batches])
    summary["levels"].append([rec.level, rec.nbatches, rec.max_rank])
np.savez(out, **save)
if decisions:
    D = O.DECISIONS
    np.savez(decisions,
             kept=np.array([r[:3] for r in D.get("kept", [])], dtype=np.int64).reshape(-1, 3),
             kept_sig=np.array([r[3:] for r in D.get("kept", [])], dtype=np.float64).reshape(-1, 2),
             created=np.array(D.get("created", []), dtype=np.int64).reshape(-1, 4),
             close=np.array(D.get("close", []), dtype=np.float64).reshape(-1, 5),
             eps_fill=fac.eps_fill, e_b=eb, e_b_raw=eb0)
print(json.dumps(summary), flush=True)
