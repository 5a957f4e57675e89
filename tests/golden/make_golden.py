"""Generate golden fixtures by importing the REFERENCE package in place.

Run here (the reference is only mounted in the build container):
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py
Writes tests/golden/<case>.npz.  Each fixture holds, for one problem:
  - a digest of the reference's H2 input (checks our problem builder),
  - norm_estimate / eps_fill,
  - the integer structure: per-level batches, r and kept per cluster,
    up_index, ncolors, csp, top_size, top pivots, per-batch fill-key sets,
  - the refined solution x (tree order), its sha256, raw and refined e_b.
"""
import hashlib
import json
import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import h2factor.factorization as fz  # noqa: E402
from h2factor.geometry import build_cluster_tree, generate_uniform_grid  # noqa: E402
from h2factor.h2core import absorb_low_rank, build_h2, matvec, orthogonalize_recompress  # noqa: E402
from h2factor.harness import PROBLEMS  # noqa: E402
from h2factor.kernels import KernelSpec, default_diag_value, make_low_rank_factor  # noqa: E402
from h2factor.solve import refined_solve, solve  # noqa: E402
from h2factor.structure import dual_tree_traversal  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = {
    "cov2d_1024": ("cov2d", 1024, {}),
    "cov2d_4096": ("cov2d", 4096, {}),
    "cov3d_2048": ("cov3d", 2048, {}),
    "laplace2d_2048": ("laplace2d", 2048, {}),
    "helmholtz3d_2048": ("helmholtz3d", 2048, {}),
    "laplace3d_4096": ("helmholtz3d", 4096, {"kappa": 0.0}),
    "osc2d_4096": ("helmholtz3d", 4096, {"dim": 2, "p0": 8, "eta": 0.9}),
    "cov3d_e8_4096": ("cov3d", 4096, {"eps_lu": 1e-8, "eps": 1e-9}),
    # round 2: config 1 itself, the config-2 / config-3 families at 16k, the
    # low-rank-update row
    "cov2d_16384": ("cov2d", 16384, {}),
    "laplace3d_16384": ("helmholtz3d", 16384, {"kappa": 0.0}),
    "cov3d_e8_16384": ("cov3d", 16384, {"eps_lu": 1e-8, "eps": 1e-9}),
    "lru_cov3d_4096": ("lru_cov3d", 4096, {}),
    "osc2d_65536": ("helmholtz3d", 65536, {"dim": 2, "p0": 8, "eta": 0.9}),
}


def h2_digest(h2):
    h = hashlib.sha256()
    for store in (h2.leaf_basis, h2.transfer, h2.coupling, h2.dense):
        for key in sorted(store):
            h.update(repr(key).encode())
            h.update(np.ascontiguousarray(store[key]).tobytes())
    return h.hexdigest()


def build(problem, n, over):
    prm = dict(PROBLEMS[problem])
    prm.update(over)
    points, counts = generate_uniform_grid(n, prm["dim"])
    tree = build_cluster_tree(points, prm["m"])
    part = dual_tree_traversal(tree, prm["eta"])
    spec = KernelSpec(family=prm["family"], dim=prm["dim"],
                      corr_length=prm["corr_length"], kappa=prm["kappa"],
                      diag_value=default_diag_value(prm["family"], 1.0 / max(counts)),
                      alpha_r=prm["alpha_r"])
    h2 = orthogonalize_recompress(build_h2(tree, part, spec, prm["p0"]), prm["eps"])
    if prm.get("lru_rank", 0) > 0:  # harness.py:185-189, seed 7
        h2 = absorb_low_rank(h2, make_low_rank_factor(n, prm["lru_rank"], 7), prm["eps"])
    return h2, prm


def capture(problem, n, over):
    h2, prm = build(problem, n, over)
    fills = []
    orig_pick = fz._pick_batch
    orig_elim = fz._eliminate_batch

    def elim_spy(state, batch, eps_fill, pool, timer):
        orig_elim(state, batch, eps_fill, pool, timer)
        fills.append(sorted(state.F))

    fz._eliminate_batch = elim_spy
    try:
        fac = fz.factorize(h2, prm["eps_lu"])
    finally:
        fz._pick_batch = orig_pick
        fz._eliminate_batch = orig_elim
    gen = np.random.Generator(np.random.Philox(7))
    x_ref = gen.standard_normal(n)
    b = matvec(h2, x_ref)
    raw = solve(fac, b)
    x = refined_solve(h2, fac, b, steps=1)
    eb = lambda v: float(np.linalg.norm(matvec(h2, v) - b) / np.linalg.norm(b))
    out = {
        "h2_digest": h2_digest(h2),
        "norm_estimate": fac.norm_estimate,
        "eps_fill": fac.eps_fill,
        "top_size": fac.top_size,
        "top_piv": fac.top_piv.astype(np.int64),
        "x": x,
        "x_raw": raw,
        "x_digest": hashlib.sha256(x.tobytes()).hexdigest(),
        "e_b_raw": eb(raw),
        "e_b": eb(x),
        "factor_bytes": fac.nbytes(),
    }
    levels = []
    for rec in fac.records:
        levels.append({
            "level": rec.level,
            "batches": rec.batches,
            "r": {int(c): int(f.r) for c, f in rec.factors.items()},
            "size": {int(c): int(s) for c, s in rec.size.items()},
            "offset": {int(c): int(o) for c, o in rec.offset.items()},
            "ncolors": rec.ncolors, "csp": rec.csp,
            "graph_degree": rec.graph_degree, "max_rank": rec.max_rank,
            "edges": {int(c): [[int(o), k, list(m.shape)] for o, k, m in f.edges]
                      for c, f in rec.factors.items()},
            "piv": {int(c): (f.piv.tolist() if f.piv is not None else None)
                    for c, f in rec.factors.items()},
        })
        out[f"up_index_{rec.level}"] = rec.up_index
    out["levels_json"] = json.dumps(levels)
    out["fills_json"] = json.dumps([[list(k) for k in f] for f in fills])
    out["params_json"] = json.dumps({"problem": problem, "n": n, **over})
    return out


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for name in names:
        problem, n, over = CASES[name]
        data = capture(problem, n, over)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **data)
        print(name, data["x_digest"][:16], f"e_b={data['e_b']:.3e}", flush=True)
