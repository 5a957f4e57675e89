"""Structure replay on the B200 (parity diagnostic).

    python scripts/replay_probe.py FAMILY N DECISIONS.npz [ORACLE.npz] [key=value ...]

Factors the operator twice through the C ABI: once with the library's own
threshold decisions, once with the CPU oracle's (kept count per cluster and
created fill blocks, recorded by scripts/oracle_big.py decisions=...).  With the
oracle's decisions the batches, ranks and fill pattern are the oracle's, so the
backward error then measures the floating-point path alone.  Prints one JSON
line per run; with ORACLE.npz also checks the replayed per-level batches and r
against the oracle's.
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2509_11152_b200 as H  # noqa: E402
from paper_2509_11152_b200 import _lib as L  # noqa: E402

fam, n, dec_path = sys.argv[1], int(sys.argv[2]), sys.argv[3]
orc_path = None
over = {}
perturb, pseed = 0.0, 1
for a in sys.argv[4:]:
    if "=" not in a:
        orc_path = a
        continue
    k, v = a.split("=")
    if k == "perturb":
        perturb = float(v)
        continue
    if k == "seed":
        pseed = int(v)
        continue
    over[k] = float(v) if "." in v or "e" in v else int(v)

tree, part, spec, h2, prm = H.build_problem(fam, n, **over)
if perturb:
    # same rounding-level perturbation as scripts/oracle_big.py perturb=... seed=...
    rng = np.random.default_rng(pseed)
    for key in sorted(h2.dense):
        blk = h2.dense[key]
        z = rng.standard_normal(blk.shape)
        if key[0] == key[1]:
            z = 0.5 * (z + z.T)
        h2.dense[key] = blk * (1.0 + perturb * z)
dec = np.load(dec_path)
orc = np.load(orc_path) if orc_path else None
x_ref = np.random.Generator(np.random.Philox(7)).standard_normal(n)
b = H.matvec(h2, x_ref)


def structure_diff(fac):
    if orc is None:
        return None
    out = []
    for rec in fac.records:
        lv = rec.level
        cl = list(rec.clusters)
        r_gpu = np.array([rec.factors[c].r for c in cl])
        bat = np.concatenate([np.array(bb) for bb in rec.batches])
        same_b = np.array_equal(bat, orc[f"L{lv}_batches"])
        out.append([lv, int(np.sum(r_gpu != orc[f"L{lv}_r"])), bool(same_b)])
    return out


for mode in ("own", "replay"):
    if mode == "replay":
        L.replay_set(dec["kept"], dec["created"])
    t0 = time.perf_counter()
    fac = H.factorize(h2, prm["eps_lu"])
    tf = time.perf_counter() - t0
    stats = L.replay_stats() if mode == "replay" else None
    L.replay_clear()
    x0 = H.solve(fac, b)
    x = H.refined_solve(h2, fac, b, steps=1)
    eb0 = float(np.linalg.norm(H.matvec(h2, x0) - b) / np.linalg.norm(b))
    eb = float(np.linalg.norm(H.matvec(h2, x) - b) / np.linalg.norm(b))
    row = {"mode": mode, "family": fam, "n": n, "over": over, "perturb": perturb, "seed": pseed,
           "fact_s": round(tf, 2), "e_b_raw": eb0, "e_b": eb,
           "oracle_e_b_raw": float(dec["e_b_raw"]), "oracle_e_b": float(dec["e_b"]),
           "top": fac.top_size, "replay": stats, "levels_r_diff_batches_equal": structure_diff(fac)}
    if orc is not None:
        row["x_vs_oracle"] = float(np.linalg.norm(x - orc["x"]) / np.linalg.norm(orc["x"]))
    print(json.dumps(row), flush=True)
    del fac
