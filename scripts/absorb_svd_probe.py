"""Isolated device QR(M^T) + Jacobi of the absorb widening residuals M of
every leaf (cov3d 2048, W rank 16) against LAPACK: orthonormality of the
left singular vectors and subspace agreement."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2509_11152_b200 import _lib as L  # noqa: E402
from paper_2509_11152_b200 import problem as P  # noqa: E402

_, _, _, h0, prm = P.build_problem("cov3d", 2048)
tree = h0.tree
w = P.make_low_rank_factor(2048, 16, 3)
for c in sorted(h0.leaf_basis):
    rows = w[tree.begin[c]:tree.end[c]]
    S = h0.leaf_basis[c]
    M = rows - S @ (S.T @ rows)
    out = []
    for qp in (0, 1):
        R, _ = L.dense_qr_r(M, qp)
        U, kept, sw, _ = L.dense_svd(R, 0.0, 0)
        U = U[:16]
        orth = np.abs(U @ U.T - np.eye(16)).max()
        perpS = np.abs(U @ S).max()
        ul = np.linalg.svd(M, full_matrices=False)[0]
        sub = np.linalg.norm(ul @ (ul.T @ U.T) - U.T)
        out.append((qp, kept, round(float(orth), 12), float(perpS), float(sub)))
    print(c, out, flush=True)
