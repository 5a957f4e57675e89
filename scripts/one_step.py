"""One factorize + refined_solve of a BASELINE config (profiling target).

    python scripts/one_step.py 2            # operator built on the device (seconds)
    python scripts/one_step.py 2 --host     # the host builder (bit-identical to the reference's)
"""
import sys

import numpy as np

sys.path.insert(0, '.')
import paper_2509_11152_b200 as H  # noqa: E402
import bench  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
cfg = bench.CONFIGS[int(args[0]) if args else 2]
if "--host" in sys.argv:
    tree, part, spec, h2, prm = H.build_problem(cfg["problem"], cfg["n"], **cfg["over"])
else:
    from paper_2509_11152_b200.construct import build_problem_device
    tree, part, spec, h2, prm = build_problem_device(cfg["problem"], cfg["n"], **cfg["over"])
b = H.matvec(h2, np.random.Generator(np.random.Philox(7)).standard_normal(h2.n))
fac = H.factorize(h2, prm["eps_lu"])
x = H.refined_solve(h2, fac, b, steps=1)
print("e_b", np.linalg.norm(H.matvec(h2, x) - b) / np.linalg.norm(b))
