"""Config 3's family (3D exponential covariance exp(-r/0.2), eps_lu = 1e-8,
eps = 1e-9) at the largest sizes one B200 holds: operator built on the
device, factorize + refined_solve timed, backward error (dev probe; the 2^20
case of BASELINE's config 3 needs the sharded factorization on 8 GPUs)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2509_11152_b200 as H  # noqa: E402
from paper_2509_11152_b200.construct import build_problem_device  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [65536, 131072]:
    tree, part, spec, h2, prm = build_problem_device("cov3d", n, eps_lu=1e-8, eps=1e-9)
    b = H.matvec(h2, np.random.Generator(np.random.Philox(7)).standard_normal(n))
    fac = H.factorize(h2, prm["eps_lu"])  # warm
    del fac
    t0 = time.perf_counter()
    fac = H.factorize(h2, prm["eps_lu"])
    x = H.refined_solve(h2, fac, b, steps=1)
    t = time.perf_counter() - t0
    eb = float(np.linalg.norm(H.matvec(h2, x) - b) / np.linalg.norm(b))
    print(json.dumps({"problem": "cov3d", "n": n, "eps_lu": 1e-8, "eps": 1e-9, "factor_plus_solve_s": t,
                      "backward_error": eb, "factor_gb": fac.nbytes() / 1e9, "top_size": fac.top_size,
                      "build_s": h2.build_seconds}), flush=True)
    del fac
