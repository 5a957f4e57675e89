"""Kernel breakdown of a 256-RHS block solve on config 2 (dev probe)."""
import sys, time, json
import numpy as np
sys.path.insert(0, '.')
import paper_2509_11152_b200 as H
from paper_2509_11152_b200 import _lib

q = int(sys.argv[1]) if len(sys.argv) > 1 else 256
tree, part, spec, h2, prm = H.build_problem("helmholtz3d", 131072, kappa=0.0)
fac = H.factorize(h2, prm["eps_lu"])
B = np.random.default_rng(1).standard_normal((h2.n, q))
H.solve_multi(fac, B)
_lib.profile_enable(True); _lib.profile_reset()
t0 = time.perf_counter()
X = H.solve_multi(fac, B)
t = time.perf_counter() - t0
prof = _lib.profile_get(); _lib.profile_enable(False)
print(json.dumps({"q": q, "wall_s": t, "kernels": {k: [round(v["seconds"], 4), v["launches"], round(v["flops"] / max(v["seconds"], 1e-12) / 1e12, 2)]
      for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["seconds"])}}))
