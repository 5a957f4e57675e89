"""Shared helpers: golden fixtures, problem construction and structural
digests used by the oracle and the GPU parity tests."""
import hashlib
import json
import os

import numpy as np
from threadpoolctl import threadpool_limits

from paper_2509_11152_b200 import problem as P

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# case -> (problem row, n, overrides); mirrors tests/golden/make_golden.py
CASES = {
    "cov2d_1024": ("cov2d", 1024, {}),
    "cov2d_4096": ("cov2d", 4096, {}),
    "cov3d_2048": ("cov3d", 2048, {}),
    "laplace2d_2048": ("laplace2d", 2048, {}),
    "helmholtz3d_2048": ("helmholtz3d", 2048, {}),
    "laplace3d_4096": ("helmholtz3d", 4096, {"kappa": 0.0}),
    "osc2d_4096": ("helmholtz3d", 4096, {"dim": 2, "p0": 8, "eta": 0.9}),
    "cov3d_e8_4096": ("cov3d", 4096, {"eps_lu": 1e-8, "eps": 1e-9}),
    "cov2d_16384": ("cov2d", 16384, {}),
    "laplace3d_16384": ("helmholtz3d", 16384, {"kappa": 0.0}),
    "cov3d_e8_16384": ("cov3d", 16384, {"eps_lu": 1e-8, "eps": 1e-9}),
    "lru_cov3d_4096": ("lru_cov3d", 4096, {}),
    "osc2d_65536": ("helmholtz3d", 65536, {"dim": 2, "p0": 8, "eta": 0.9}),
}

_cache = {}


def load(case):
    with np.load(os.path.join(GOLDEN, f"{case}.npz")) as z:
        d = {k: z[k] for k in z.files}
    d["levels"] = json.loads(str(d.pop("levels_json")))
    d["fills"] = json.loads(str(d.pop("fills_json")))
    d["params"] = json.loads(str(d.pop("params_json")))
    return d


def problem(case):
    if case not in _cache:
        name, n, over = CASES[case]
        _cache[case] = P.build_problem(name, n, **over)
    return _cache[case]


def h2_digest(h2):
    h = hashlib.sha256()
    for store in (h2.leaf_basis, h2.transfer, h2.coupling, h2.dense):
        for key in sorted(store):
            h.update(repr(key).encode())
            h.update(np.ascontiguousarray(store[key]).tobytes())
    return h.hexdigest()


def rhs(h2, matvec, seed=7):
    x_ref = np.random.Generator(np.random.Philox(seed)).standard_normal(h2.n)
    return matvec(h2, x_ref)


def structure_of(fac):
    """Integer structure of a factorization in the golden's JSON layout."""
    out = []
    for rec in fac.records:
        out.append({
            "level": int(rec.level),
            "batches": [[int(c) for c in b] for b in rec.batches],
            "r": {str(int(c)): int(f.r) for c, f in rec.factors.items()},
            "size": {str(int(c)): int(s) for c, s in rec.size.items()},
            "ncolors": int(rec.ncolors), "csp": int(rec.csp),
            "graph_degree": int(rec.graph_degree), "max_rank": int(rec.max_rank),
        })
    return out


def golden_structure(g):
    return [{k: lv[k] for k in ("level", "batches", "r", "size", "ncolors", "csp",
                                "graph_degree", "max_rank")}
            for lv in g["levels"]]


def one_thread():
    return threadpool_limits(1)
