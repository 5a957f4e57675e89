"""Capture upper-level augmentation inputs (V, fill row) of a 3D Laplace 16384
factorization from the oracle, for scripts/jacobi_sweep_study.py."""
import sys, numpy as np, pickle
sys.path.insert(0, '/root/repo')
from threadpoolctl import threadpool_limits
from oracle import h2_oracle as O
from paper_2509_11152_b200 import problem as P
tree, part, spec, h2, prm = P.build_problem("helmholtz3d", 16384, kappa=0.0)
cap = []
orig = O.augment
def aug(v, fill, eps_fill):
    if fill.shape[1] >= v.shape[0] and v.shape[0] - v.shape[1] >= 150 and len(cap) < 12:
        cap.append((v.copy(), fill.copy(), eps_fill))
    return orig(v, fill, eps_fill)
O.augment = aug
with threadpool_limits(8):
    O.factorize(h2, prm["eps_lu"])
pickle.dump(cap, open('/tmp/jac/cap.pkl', 'wb'))
print(len(cap), [(c[0].shape, c[1].shape) for c in cap])
