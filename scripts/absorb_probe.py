"""Device absorb_low_rank diagnostic: operator error of the widened (eps=0,
no recompression) and recompressed device operators against the exact
A x + W W^T x, next to the host absorb_low_rank's."""
import copy
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2509_11152_b200 as H  # noqa: E402
from paper_2509_11152_b200 import problem as P  # noqa: E402
from paper_2509_11152_b200.construct import absorb_low_rank_device  # noqa: E402

out = {}
for name, n, r, seed in [("cov3d", 2048, 16, 3), ("cov2d", 4096, 8, 1)]:
    _, _, _, h0, prm = P.build_problem(name, n)
    w = P.make_low_rank_factor(n, r, seed)
    hh = P.absorb_low_rank(copy.deepcopy(h0), w, prm["eps"])  # before h0 caches a device handle
    x = np.random.default_rng(5).standard_normal(n)
    exact = H.matvec(h0, x) + w @ (w.T @ x)
    d0 = absorb_low_rank_device(h0, w, 0.0)
    d1 = absorb_low_rank_device(h0, w, prm["eps"])
    rel = lambda y: float(np.linalg.norm(y - exact) / np.linalg.norm(exact))  # noqa: E731
    out[f"{name}_{n}"] = {"host_absorb": rel(H.matvec(hh, x)), "device_widened_only": rel(H.matvec(d0, x)),
                          "device_absorb": rel(H.matvec(d1, x)),
                          "ranks_host": [int(hh.rank.get(c, -1)) for c in range(len(h0.tree.parent))],
                          "ranks_dev_widened": [int(d0.rank.get(c, -1)) for c in range(len(h0.tree.parent))],
                          "ranks_dev": [int(d1.rank.get(c, -1)) for c in range(len(h0.tree.parent))]}
    print(name, n, {k: v for k, v in out[f"{name}_{n}"].items() if not k.startswith("ranks")}, flush=True)
json.dump(out, open("gpurun_out/absorb_probe.json", "w"))
