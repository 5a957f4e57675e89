"""Host-side margins of the absorb_low_rank recompression: how close each
singular value sits to the eps * sigma_0 cut (tests/test_gpu_construct.py)."""
import copy, numpy as np
from paper_2509_11152_b200 import problem as P
orig_svd = np.linalg.svd
log = []
def svd(a, full_matrices=True, **kw):
    u, s, v = orig_svd(a, full_matrices=full_matrices, **kw)
    log.append(s.copy())
    return u, s, v
_, _, _, h0, prm = P.build_problem("cov3d", 2048)
w = P.make_low_rank_factor(2048, 16, 3)
np.linalg.svd = svd
hh = P.absorb_low_rank(copy.deepcopy(h0), w, prm["eps"])
np.linalg.svd = orig_svd
# margins: for each svd, min |log10(sig/cut)| for cut candidates eps*sig0 and 1e-12 scale unknown -> report eps one
worst = []
for s in log:
    if s.size == 0: continue
    cut = prm["eps"] * s[0]
    r = np.abs(np.log10(np.maximum(s, 1e-300) / cut))
    worst.append(r.min())
worst = np.array(worst)
print(len(log), "svds; eps", prm["eps"], "closest |log10(sig/cut)| sorted:", np.sort(worst)[:10])
# range basis: values near 1e-12 * scale relative to sig[0]
for s in log[:]:
    pass
