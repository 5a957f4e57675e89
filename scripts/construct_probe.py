"""Device H2 construction vs the host builder (dev diagnostic, GPU box).

    python scripts/construct_probe.py cov2d:4096 helmholtz3d:16384:kappa=0 ...

Per case: host build time (problem.build_problem), device build time
(construct.build_problem_device), rank agreement, matvec difference between
the two operators, dense-kernel error of both on sampled rows (n <= 16384),
and the factor + refined-solve backward error on each operator.
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2509_11152_b200 as H  # noqa: E402
from paper_2509_11152_b200 import problem as P  # noqa: E402
from paper_2509_11152_b200.construct import build_problem_device  # noqa: E402


def parse(arg):
    parts = arg.split(":")
    name, n = parts[0], int(parts[1])
    over = {}
    for kv in parts[2:]:
        k, v = kv.split("=")
        over[k] = float(v) if ("." in v or "e" in v) else int(v)
    return name, n, over


def eb(h2, fac, b):
    x = H.refined_solve(h2, fac, b, steps=1)
    return float(np.linalg.norm(H.matvec(h2, x) - b) / np.linalg.norm(b))


def main():
    factor = "--no-factor" not in sys.argv
    host = "--no-host" not in sys.argv
    for arg in [a for a in sys.argv[1:] if not a.startswith("--")]:
        name, n, over = parse(arg)
        out = {"case": arg}
        tree, part, spec, hd, prm = build_problem_device(name, n, **over)
        H.matvec(hd, np.ones(n))  # warm
        t0 = time.perf_counter()
        tree, part, spec, hd, prm = build_problem_device(name, n, **over)
        out["device_build_s"] = time.perf_counter() - t0
        out["device_seconds"] = hd.build_seconds
        out["device_nbytes"] = hd._h2f_built.nbytes
        kd = np.array([hd.rank.get(c, -1) for c in range(len(tree.parent))])
        out["kmax_device"] = int(kd.max())
        rng = np.random.default_rng(0)
        x = rng.standard_normal(n)
        yd = H.matvec(hd, x)
        if host:
            t0 = time.perf_counter()
            _, _, _, hh, _ = P.build_problem(name, n, **over)
            out["host_build_s"] = time.perf_counter() - t0
            kh = np.array([hh.rank.get(c, -1) for c in range(len(tree.parent))])
            diff = kd - kh
            out["rank_equal_frac"] = float(np.mean(diff == 0))
            out["rank_absdiff_max"] = int(np.abs(diff).max())
            out["kmax_host"] = int(kh.max())
            yh = H.matvec(hh, x)
            out["matvec_rel_diff"] = float(np.linalg.norm(yd - yh) / np.linalg.norm(yh))
            if n <= 16384:
                rows = rng.choice(n, size=min(n, 256), replace=False)
                K = P.entry_block(spec, tree.points, rows, np.arange(n))
                ex = K @ x
                out["dense_err_device"] = float(np.linalg.norm(yd[rows] - ex) / np.linalg.norm(ex))
                out["dense_err_host"] = float(np.linalg.norm(yh[rows] - ex) / np.linalg.norm(ex))
        if factor:
            xr = P.rhs_for(hd)
            b = H.matvec(hd, xr)
            fac = H.factorize(hd, prm["eps_lu"])
            out["e_b_device_op"] = eb(hd, fac, b)
            if host:
                bh = H.matvec(hh, xr)
                fh = H.factorize(hh, prm["eps_lu"])
                out["e_b_host_op"] = eb(hh, fh, bh)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
