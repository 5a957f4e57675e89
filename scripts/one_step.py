"""One factorize + refined_solve of a BASELINE config (profiling target)."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2509_11152_b200 as H
import bench

cfg = bench.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
tree, part, spec, h2, prm = H.build_problem(cfg["problem"], cfg["n"], **cfg["over"])
b = H.matvec(h2, np.random.Generator(np.random.Philox(7)).standard_normal(h2.n))
fac = H.factorize(h2, prm["eps_lu"])
x = H.refined_solve(h2, fac, b, steps=1)
print("e_b", np.linalg.norm(H.matvec(h2, x) - b) / np.linalg.norm(b))
