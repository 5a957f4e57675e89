"""Device harness: the reference's measured pipeline
`harness.run(config)` (/root/reference/pkg/src/h2factor/harness.py:197-249)
with the factorization and the refined solve on the B200 path.

`run(problem, n, **overrides)` builds the operator on the host exactly like
the reference (grid, KD tree, dual-tree partition, Chebyshev H2,
recompression -- problem.py), factors it, solves for b = A x_ref with
x_ref ~ Philox(seed) normal, and returns a report with the reference
RunReport's keys (version, config, n, e_b, solution_digest, h2_bytes,
factor_bytes, kmax_construction, kmax_factorization, csp_max, timings,
phases, levels, ranks; `solution` omitted unless asked for).  Timings are
host wall clock around the public API calls, as in the reference; the
factorization's `phases` come from CUDA events on the library stream.

    python -m paper_2509_11152_b200.harness cov2d 16384 [key=value ...]
"""
from __future__ import annotations

import hashlib
import json
import sys
import time

import numpy as np

from . import __version__
from .factorization import factorize
from .h2core import matvec
from .problem import build_problem, h2_nbytes
from .solve import refined_solve

# harness.py:74-83 of the reference
PHASE_LABELS = {
    "norm": "norm_estimate",
    "extract": "block_extract",
    "color": "coloring",
    "augment": "basis_augmentation",
    "project": "projection",
    "partial_lu": "partial_lu",
    "transition": "level_transition",
    "top": "top_solve",
}


def run(problem, n, seed=7, refine_steps=1, keep_solution=False, **overrides):
    t0 = time.perf_counter()
    tree, part, spec, h2, prm = build_problem(problem, n, **overrides)
    t_build = time.perf_counter() - t0
    timings = {"construction_and_compression": t_build}

    t0 = time.perf_counter()
    fac = factorize(h2, prm["eps_lu"])
    timings["factorization"] = time.perf_counter() - t0

    x_ref = np.random.Generator(np.random.Philox(seed)).standard_normal(h2.n)
    b = matvec(h2, x_ref)
    t0 = time.perf_counter()
    x = refined_solve(h2, fac, b, steps=refine_steps)
    timings["solve"] = time.perf_counter() - t0
    e_b = float(np.linalg.norm(matvec(h2, x) - b) / np.linalg.norm(b))

    phases = {"construction_and_compression": t_build}
    for key, label in PHASE_LABELS.items():
        if key in fac.phase_seconds:
            phases[label] = fac.phase_seconds[key]
    phases["solve"] = timings["solve"]
    levels = [{"level": r.level, "time_s": r.time_s, "csp": r.csp, "max_rank": r.max_rank} for r in fac.records]
    report = {
        "version": __version__,
        "device": "cuda",
        "config": {"problem": problem, "n": n, "seed": seed, "refine_steps": refine_steps, **prm},
        "n": int(h2.n),
        "e_b": e_b,
        "solution_digest": hashlib.sha256(x.tobytes()).hexdigest(),
        "h2_bytes": int(h2_nbytes(h2)),
        "factor_bytes": int(fac.nbytes()),
        "kmax_construction": int(max(h2.rank.values())) if h2.rank else 0,
        "kmax_factorization": int(fac.max_rank()),
        "csp_max": int(max((r.csp for r in fac.records), default=0)),
        "timings": timings,
        "phases": phases,
        "levels": levels,
        "ranks": [r.max_rank for r in fac.records],
    }
    if keep_solution:
        report["solution"] = x
    return report


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    if len(argv) < 2:
        print(__doc__)
        return 2
    over = {}
    for a in argv[2:]:
        k, v = a.split("=")
        over[k] = float(v) if any(ch in v for ch in ".e") else int(v)
    print(json.dumps(run(argv[0], int(argv[1]), **over)))
    return 0


if __name__ == "__main__":
    sys.exit(main())
