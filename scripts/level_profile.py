"""Per-level device kernel seconds and host section times of one config-2
factorization (H2F_LEVEL_PROF=1 with the profiler on; stderr), operator
built on the device (construct.py) to skip the 97 s host builder."""
import os
import sys
import time

sys.path.insert(0, ".")
os.environ.setdefault("H2F_LEVEL_PROF", "1")
import paper_2509_11152_b200 as H  # noqa: E402
from paper_2509_11152_b200 import _lib  # noqa: E402
from paper_2509_11152_b200.construct import build_problem_device  # noqa: E402

name, n = (sys.argv[1], int(sys.argv[2])) if len(sys.argv) > 2 else ("helmholtz3d", 131072)
tree, part, spec, h2, prm = build_problem_device(name, n, kappa=0.0)
fac = H.factorize(h2, prm["eps_lu"])  # warm
del fac
t0 = time.perf_counter()
fac = H.factorize(h2, prm["eps_lu"])
print("factorize (profiler off) %.3f s" % (time.perf_counter() - t0), flush=True)
del fac
_lib.profile_enable(True)
_lib.profile_reset()
t0 = time.perf_counter()
fac = H.factorize(h2, prm["eps_lu"])
print("factorize (profiler on) %.3f s" % (time.perf_counter() - t0), flush=True)
prof = _lib.profile_get()
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["seconds"])[:14]:
    print("  %-20s %8.4f s  %6d launches" % (k, v["seconds"], v["launches"]))
for r in fac.records:
    print("level", r.level, "clusters", len(r.clusters), "batches", r.nbatches,
          "mean batch", round(len(r.clusters) / max(r.nbatches, 1), 2), "time_s", round(r.time_s, 4))
