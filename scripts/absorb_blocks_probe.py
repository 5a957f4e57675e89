"""Block-level check of the device absorb_low_rank widening (eps = 0):
dense blocks, basis orthonormality / reproduction of W, and admissible
blocks U_s C U_t^T against the host operator's blocks + W_s W_t^T."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2509_11152_b200 import problem as P  # noqa: E402
from paper_2509_11152_b200.construct import absorb_low_rank_device, export_blocks  # noqa: E402

_, _, _, h0, prm = P.build_problem("cov3d", 2048)
tree = h0.tree
w = P.make_low_rank_factor(2048, 16, 3)
d0 = absorb_low_rank_device(h0, w, 0.0)
B = export_blocks(d0)
Wr = lambda c: w[tree.begin[c]:tree.end[c]]  # noqa: E731

worst = 0
for (s, t), blk in B["dense"].items():
    ref = h0.dense[(s, t)] + Wr(s) @ Wr(t).T
    worst = max(worst, np.abs(blk - ref).max() / np.abs(ref).max())
print("dense max rel", worst)


def full_basis(store, c):
    if c in store["leaf_basis"]:
        return store["leaf_basis"][c]
    a, b = tree.children(c)
    Ua, Ub = full_basis(store, a), full_basis(store, b)
    Ta, Tb = store["transfer"][a], store["transfer"][b]
    return np.vstack([Ua @ Ta, Ub @ Tb])


h0s = {"leaf_basis": h0.leaf_basis, "transfer": h0.transfer}
bad = []
for c in sorted(d0.rank):
    U = full_basis(B, c)
    orth = np.abs(U.T @ U - np.eye(U.shape[1])).max()
    rep = np.linalg.norm(Wr(c) - U @ (U.T @ Wr(c))) / np.linalg.norm(Wr(c))
    if orth > 1e-10 or rep > 1e-10:
        bad.append((c, int(tree.level[c]), U.shape, float(orth), float(rep)))
print("basis problems (cluster, level, shape, orth, W repro):", bad[:12], len(bad))
worst = []
for (s, t), C in B["coupling"].items():
    Us, Ut = full_basis(B, s), full_basis(B, t)
    U0s, U0t = full_basis(h0s, s), full_basis(h0s, t)
    ref = U0s @ h0.coupling[(s, t)] @ U0t.T + Wr(s) @ Wr(t).T
    got = Us @ C @ Ut.T
    worst.append((float(np.abs(got - ref).max() / np.abs(ref).max()), s, t, int(tree.level[s])))
worst.sort(reverse=True)
print("worst coupling blocks (rel, s, t, level):", worst[:8])
