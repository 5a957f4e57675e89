"""Micro-benchmark of the per-cluster dense kernels on config-2-like shapes
(dev aid; shapes from the augmentation log of 3D Laplace N=131072)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2509_11152_b200 import _lib  # noqa: E402


def graded(m, n, decay, seed):
    rng = np.random.Generator(np.random.Philox(seed))
    u, _ = np.linalg.qr(rng.standard_normal((m, m)))
    v, _ = np.linalg.qr(rng.standard_normal((n, m)))
    sig = 10.0 ** (-decay * np.arange(m) / m)
    return (u * sig) @ v.T, sig


what = sys.argv[1:] or ["svd", "qr", "cmp"]
if "svd" in what:
    for n in [118, 219, 358, 600, 844, 1170]:
        Y, sig = graded(n, 2 * n, 14.0, n)
        R = np.linalg.qr(Y.T, mode="r")
        thresh = sig[int(0.7 * n)]
        for path in ([0] if n <= 144 else []) + [1, 2]:
            _lib.dense_svd(R, thresh, path)
            U, kept, sweeps, ms = _lib.dense_svd(R, thresh, path)
            print(f"svd n={n:5d} path={path} kept={kept:4d} sweeps={sweeps:3d} {ms:9.3f} ms", flush=True)
if "qr" in what:
    for n, wf in [(52, 7800), (118, 13800), (219, 20400), (358, 23900), (600, 15000), (844, 4400)]:
        Y, _ = graded(n, wf, 10.0, n)
        for path in ([0] if n <= 144 else []) + [1]:
            _lib.dense_qr_r(Y, path)
            R, ms = _lib.dense_qr_r(Y, path)
            print(f"qr  n={n:5d} wf={wf:6d} path={path} {ms:9.3f} ms", flush=True)
if "cmp" in what:
    for s, kt in [(106, 88), (178, 138), (276, 208), (416, 323), (646, 440), (880, 581)]:
        rng = np.random.Generator(np.random.Philox(s))
        b = np.linalg.qr(rng.standard_normal((s, kt)))[0]
        for path in [0, 1]:
            _lib.dense_complement(np.ascontiguousarray(b.T), path)
            Q, ms = _lib.dense_complement(np.ascontiguousarray(b.T), path)
            print(f"cmp s={s:5d} kt={kt:5d} path={path} {ms:9.3f} ms", flush=True)
