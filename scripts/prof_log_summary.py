"""Summarise an H2F_PROF_LOG per-launch log: per kernel, time-weighted
achieved rate binned by launch size (dev aid)."""
import collections, sys

rows = [l.split() for l in open(sys.argv[1])]
want = sys.argv[2] if len(sys.argv) > 2 else "gemm_schur"
bins = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])  # n, ms, flops, bytes
for k, f, b, u, ms in rows:
    if k != want:
        continue
    f, b, u, ms = float(f), float(b), float(u), float(ms)
    key = 10 ** int(len(str(int(max(u, 1)))) - 1)  # decade of tile count
    e = bins[key]
    e[0] += 1; e[1] += ms; e[2] += f; e[3] += b
tot = sum(e[1] for e in bins.values())
print(f"{want}: {tot/1e3:.3f} s total")
for key in sorted(bins):
    n, ms, f, b = bins[key]
    print(f"tiles ~{key:>8d}: {n:5d} launches {ms/1e3:8.3f} s ({100*ms/tot:5.1f}%)  {f/ms/1e9:7.2f} TF/s  {b/ms/1e6:7.1f} GB/s  AI {f/max(b,1):.1f}")
