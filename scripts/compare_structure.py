"""Compare the per-level structure of two factorizations saved as npz by
scripts/oracle_big.py (CPU oracle) and scripts/draws_probe.py save=... (B200):
elimination order, batch lengths and redundant counts r per cluster, level by
level from the leaf.  Dev aid: python scripts/compare_structure.py A.npz B.npz"""
import sys

import numpy as np

a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
levels = sorted({int(k[1:].split('_')[0]) for k in a.files if k.startswith('L')}, reverse=True)
for lv in levels:
    ca, cb = a[f"L{lv}_batches"], b[f"L{lv}_batches"]
    ra = dict(zip(a[f"L{lv}_clusters"], a[f"L{lv}_r"]))
    rb = dict(zip(b[f"L{lv}_clusters"], b[f"L{lv}_r"]))
    sa = dict(zip(a[f"L{lv}_clusters"], a[f"L{lv}_size"]))
    sb = dict(zip(b[f"L{lv}_clusters"], b[f"L{lv}_size"]))
    n = min(len(ca), len(cb))
    first_order = next((i for i in range(n) if ca[i] != cb[i]), None)
    order = list(ca)
    first_r = next((i for i, c in enumerate(order) if ra[c] != rb.get(c)), None)
    nr = sum(ra[c] != rb.get(c) for c in order)
    skel_a = sum(sa[c] - ra[c] for c in order)
    skel_b = sum(sb[c] - rb[c] for c in order)
    print(f"L{lv}: clusters {len(ca)} batches {len(a[f'L{lv}_blen'])}/{len(b[f'L{lv}_blen'])} "
          f"order diverges at {first_order} r differs at {first_r} ({nr} differ) "
          f"sum skeleton {skel_a}/{skel_b} sum size {sum(sa.values())}/{sum(sb.values())}")
xa, xb = a["x"], b["x"]
print("solution rel diff", float(np.linalg.norm(xa - xb) / np.linalg.norm(xa)))
