"""Offline one-sided Jacobi sweep counts (numpy, the GPU rotation/convergence
rule) on R of captured fill rows: as computed, with a second QR, with rows
presorted, and with a column-pivoted QR."""
import sys, numpy as np, pickle, scipy.linalg as sl
def rr_pairs(m):
    mm = m + (m & 1); idx = list(range(mm))
    for st in range(mm - 1):
        pairs = [(idx[i], idx[mm - 1 - i]) for i in range(mm // 2)]
        yield [(p, q) for p, q in pairs if p < m and q < m]
        idx = [idx[0]] + [idx[-1]] + idx[1:-1]
def jacobi_sweeps(A, tol_cos=1e-7, maxs=60):
    A = A.copy(); m, n = A.shape
    for sw in range(1, maxs + 1):
        mx = 0.0
        for pairs in rr_pairs(m):
            p = np.array([a for a, b in pairs]); q = np.array([b for a, b in pairs])
            ap, aq = A[p], A[q]
            al = (ap * ap).sum(1); be = (aq * aq).sum(1); ga = (ap * aq).sum(1)
            den = np.sqrt(al * be); cs = np.where(den > 0, np.abs(ga) / np.maximum(den, 1e-300), 0)
            mx = max(mx, cs.max() if len(cs) else 0)
            rot = cs > 2.2e-16 * np.sqrt(n)
            if not rot.any(): continue
            z = (be - al) / (2 * np.where(rot, ga, 1))
            t = np.sign(z) / (np.abs(z) + np.sqrt(1 + z * z)); t = np.where(z == 0, 1.0, t)
            c = 1 / np.sqrt(1 + t * t); s = c * t
            c = np.where(rot, c, 1.0); s = np.where(rot, s, 0.0)
            A[p] = c[:, None] * ap - s[:, None] * aq
            A[q] = s[:, None] * ap + c[:, None] * aq
        if mx <= tol_cos:
            return sw, A
    return maxs, A
cap = pickle.load(open('/tmp/jac/cap.pkl', 'rb'))
for v, fill, eps_fill in cap:
    s, k = v.shape
    Qv = np.linalg.qr(v, mode='complete')[0]
    Vp = Qv[:, k:]
    Z = Vp.T @ fill
    n = Z.shape[0]
    R = np.linalg.qr(Z.T, mode='r')
    R = np.triu(R[:n])
    sw0, _ = jacobi_sweeps(R)
    R1 = np.linalg.qr(R.T, mode='r')           # R^T = Q1 R1
    sw1, _ = jacobi_sweeps(np.triu(R1).T)      # rows of R1^T
    # sorted rows by norm
    o = np.argsort(-np.linalg.norm(R, axis=1))
    sw2, _ = jacobi_sweeps(R[o])
    # pivoted first QR (Drmac)
    _, Rp, piv = sl.qr(Z.T, mode='economic', pivoting=True)
    R1p = np.linalg.qr(Rp.T, mode='r')
    sw3, _ = jacobi_sweeps(np.triu(R1p).T)
    sig = np.linalg.svd(Z, compute_uv=False)
    drop = 0.01 * eps_fill
    print(f"n={n} wf={Z.shape[1]} kept={(sig >= drop).sum()} sig0/drop={sig[0]/drop:.1e}  sweeps: R={sw0} R1^T={sw1} sortedR={sw2} pivR1^T={sw3}", flush=True)
