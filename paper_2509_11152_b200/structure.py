"""Multi-level graph colouring primitives (structure.py:127-167 of the
reference).  greedy_coloring runs the same C++ routine the factorization
uses for each level's schedule, through the C ABI."""
from __future__ import annotations

import numpy as np

from . import _lib as L

__all__ = ["level_graph", "greedy_coloring", "color_groups", "sparsity_constant"]


def level_graph(clusters, pairs):
    """Adjacency over clusters induced by canonical pairs (self edges
    dropped): {cluster: sorted neighbour array}."""
    neigh = {int(c): set() for c in clusters}
    for s, t in pairs:
        if s != t:
            neigh[int(s)].add(int(t))
            neigh[int(t)].add(int(s))
    return {c: np.array(sorted(v), dtype=np.int64) for c, v in neigh.items()}


def greedy_coloring(adjacency):
    """Colour in ascending id order, smallest colour unused by coloured
    neighbours.  Computed by libh2f (h2f_greedy_coloring)."""
    ids = np.array(sorted(adjacency), dtype=np.int64)
    pairs = [(int(c), int(j)) for c in ids for j in adjacency[c] if c < j]
    flat = np.array(pairs, dtype=np.int64).reshape(-1)
    colors = np.empty(max(len(ids), 1), dtype=np.int32)
    ncol = np.zeros(1, dtype=np.int32)
    deg = np.zeros(1, dtype=np.int32)
    L.check(L.lib().h2f_greedy_coloring(len(ids), L.ptr(ids, L.i64p), len(pairs),
                                        L.ptr(flat, L.i64p), L.ptr(colors, L.i32p),
                                        L.ptr(ncol, L.i32p), L.ptr(deg, L.i32p)))
    return {int(c): int(k) for c, k in zip(ids, colors[:len(ids)])}


def color_groups(color):
    """Colours as lists of cluster ids, ascending within each colour."""
    ncol = max(color.values()) + 1 if color else 0
    groups = [[] for _ in range(ncol)]
    for c in sorted(color):
        groups[color[c]].append(c)
    return groups


def sparsity_constant(partition, level):
    """Max number of dense blocks in any block row of `level`."""
    cnt = {}
    dense = set(partition.inadmissible_inner[level]) | set(partition.inadmissible_leaves[level])
    for s, t in dense:
        cnt[s] = cnt.get(s, 0) + 1
        if t != s:
            cnt[t] = cnt.get(t, 0) + 1
    return max(cnt.values()) if cnt else 0
