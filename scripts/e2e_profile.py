"""cProfile of the public-API end-to-end path of the config-2 bench (e2e):
operator upload, factorize, refined_solve with host buffers (dev probe)."""
import cProfile
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2509_11152_b200 as H  # noqa: E402

tree, part, spec, h2, prm = H.build_problem("helmholtz3d", 131072, kappa=0.0)
b = H.matvec(h2, np.random.Generator(np.random.Philox(7)).standard_normal(h2.n))
fac = H.factorize(h2, prm["eps_lu"])  # warm
del fac
object.__setattr__(h2, "_h2f_device", None)
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
fac = H.factorize(h2, prm["eps_lu"])
x = H.refined_solve(h2, fac, b, steps=1)
pr.disable()
print("e2e", time.perf_counter() - t0)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
