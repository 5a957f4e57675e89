"""factorize() on the B200 and the factor objects it returns.

Drop-in for /root/reference/pkg/src/h2factor/factorization.py:
  factorize(h2, eps_lu, threads=1, norm_estimate=None) -> H2Factorization
  FactorizationError, PIVOT_RTOL, FILL_DROP_FACTOR,
  H2Factorization / LevelRecord / ClusterFactor with the same fields.

The whole level loop runs inside libh2f (C++ scheduler + sm_100a kernels);
this module only packs the input and exposes the factor.  Integer structure
(batches, r, offsets, up_index, colouring statistics) is exported eagerly;
floating-point factor blocks (q, lu, edges, top_lu) are copied from the
device lazily on first access.  `threads` is accepted for API parity: the
reference's thread pool (parallel.py) is replaced by device batching.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .h2core import device_matrix, power_start

__all__ = ["FactorizationError", "H2Factorization", "LevelRecord", "ClusterFactor", "factorize",
           "PIVOT_RTOL", "FILL_DROP_FACTOR", "PHASES"]

PIVOT_RTOL = 1e-14        # factorization.py:47
FILL_DROP_FACTOR = 1e-2   # factorization.py:55
PHASES = ("norm", "extract", "color", "augment", "project", "partial_lu", "transition", "top")
_KINDS = ("self", "full", "skel")


class FactorizationError(RuntimeError):
    """A diagonal block of redundant coordinates could not be eliminated
    (factorization.py:58-59)."""


class _Handle:
    def __init__(self, ptr, matrix):
        self.ptr = ptr
        self.matrix = matrix  # keeps the device operator alive

    def __del__(self):
        if self.ptr is not None and self.ptr.value and L._lib is not None:
            L._lib.h2f_factor_destroy(self.ptr)
            self.ptr = None


class ClusterFactor:
    """Per-cluster elimination data (factorization.py:130-147); arrays are
    fetched from the device on first access."""

    __slots__ = ("_h", "_rec", "cluster", "level", "r", "size", "_q", "_lu", "_piv", "_edges", "_nedges")

    def __init__(self, handle, rec, cluster, level, size, r, nedges):
        self._h, self._rec = handle, rec
        self.cluster, self.level, self.size, self.r = cluster, level, size, r
        self._nedges = nedges
        self._q = self._lu = self._piv = self._edges = None

    def _fetch(self):
        s, r, ne = self.size, self.r, self._nedges
        q = np.empty((s, s))
        lu = np.empty((r, r)) if r else None
        piv = np.empty(r, dtype=np.int32) if r else None
        other = np.empty(max(ne, 1), dtype=np.int64)
        kind = np.empty(max(ne, 1), dtype=np.int32)
        width = np.empty(max(ne, 1), dtype=np.int64)
        L.check(L.lib().h2f_factor_cluster_arrays(
            self._h.ptr, self._rec, self.cluster, L.ptr(q),
            L.ptr(lu) if r else None, L.ptr(piv, L.i32p) if r else None,
            L.ptr(other, L.i64p), L.ptr(kind, L.i32p), L.ptr(width, L.i64p)))
        edges = []
        for e in range(ne):
            mat = np.empty((r, int(width[e])))
            L.check(L.lib().h2f_factor_cluster_edge(self._h.ptr, self._rec, self.cluster, e, L.ptr(mat)))
            edges.append((int(other[e]), _KINDS[kind[e]], mat))
        self._q = q
        self._lu = np.asfortranarray(lu) if r else None  # scipy lu_factor layout
        self._piv = piv
        self._edges = edges

    @property
    def q(self):
        if self._q is None:
            self._fetch()
        return self._q

    @property
    def lu(self):
        if self._q is None:
            self._fetch()
        return self._lu

    @property
    def piv(self):
        if self._q is None:
            self._fetch()
        return self._piv

    @property
    def edges(self):
        if self._q is None:
            self._fetch()
        return self._edges


class LevelRecord:
    """factorization.py:150-164."""

    def __init__(self, handle, idx):
        info = L.LevelInfo()
        L.check(L.lib().h2f_factor_level_info(handle.ptr, idx, C.byref(info)))
        nc, nbt = info.num_clusters, info.num_batches
        clusters = np.empty(nc, dtype=np.int64)
        offs = np.empty(nc, dtype=np.int64)
        sizes = np.empty(nc, dtype=np.int64)
        bptr = np.empty(nbt + 1, dtype=np.int64)
        bids = np.empty(max(info.batch_entries, 1), dtype=np.int64)
        up = np.empty(info.up_size, dtype=np.int64)
        L.check(L.lib().h2f_factor_level_arrays(
            handle.ptr, idx, L.ptr(clusters, L.i64p), L.ptr(offs, L.i64p), L.ptr(sizes, L.i64p),
            L.ptr(bptr, L.i64p), L.ptr(bids, L.i64p), L.ptr(up, L.i64p)))
        self.level = info.level
        self.clusters = [int(c) for c in clusters]
        self.offset = {int(c): int(o) for c, o in zip(clusters, offs)}
        self.size = {int(c): int(s) for c, s in zip(clusters, sizes)}
        self.batches = [[int(c) for c in bids[bptr[b]:bptr[b + 1]]] for b in range(nbt)]
        self.up_index = up
        self.csp = info.csp
        self.ncolors = info.ncolors
        self.nbatches = nbt
        self.graph_degree = info.graph_degree
        self.max_rank = info.max_rank
        self.time_s = info.time_s
        self._h, self._idx = handle, idx
        factors = {}
        for c in self.clusters:
            ci = L.ClusterInfo()
            L.check(L.lib().h2f_factor_cluster_info(handle.ptr, idx, c, C.byref(ci)))
            factors[c] = ClusterFactor(handle, idx, c, self.level, ci.size, ci.r, ci.num_edges)
        self.factors = factors

    def fill_events(self):
        """(initial fill keys, [(batch, (a, b)), ...] created in order)
        (factorization.py:502-505, 573-588)."""
        ni, nc = C.c_int64(), C.c_int64()
        L.check(L.lib().h2f_factor_level_fills(self._h.ptr, self._idx, C.byref(ni), None, C.byref(nc), None))
        init = np.empty((max(ni.value, 1), 2), dtype=np.int64)
        made = np.empty((max(nc.value, 1), 3), dtype=np.int64)
        L.check(L.lib().h2f_factor_level_fills(self._h.ptr, self._idx, C.byref(ni), L.ptr(init, L.i64p),
                                               C.byref(nc), L.ptr(made, L.i64p)))
        return ([(int(a), int(b)) for a, b in init[:ni.value]],
                [(int(t), (int(a), int(b))) for t, a, b in made[:nc.value]])

    def fill_keys_after_batches(self):
        """Sorted F-key set after every batch of this level."""
        init, made = self.fill_events()
        keys, out, i = set(init), [], 0
        for b in range(self.nbatches):
            while i < len(made) and made[i][0] == b:
                keys.add(made[i][1])
                i += 1
            out.append(sorted(keys))
        return out


class H2Factorization:
    """factorization.py:167-193.  The factor itself stays on the device."""

    def __init__(self, tree, handle):
        info = L.FactorInfo()
        L.check(L.lib().h2f_factor_info_get(handle.ptr, C.byref(info)))
        self._h = handle
        self.tree = tree
        self.n = int(info.n)
        self.top_level = None if info.top_level < 0 else int(info.top_level)
        self.top_size = int(info.top_size)
        self.eps_lu = float(info.eps_lu)
        self.eps_fill = float(info.eps_fill)
        self.norm_estimate = float(info.norm_estimate)
        self.phase_seconds = {k: float(info.phase_seconds[i]) for i, k in enumerate(PHASES)}
        self._nbytes = int(info.nbytes)
        self.records = [LevelRecord(handle, i) for i in range(info.num_records)]
        self._top = None

    def _fetch_top(self):
        n = self.top_size
        lu = np.empty((n, n))
        piv = np.empty(n, dtype=np.int32)
        L.check(L.lib().h2f_factor_top(self._h.ptr, L.ptr(lu), L.ptr(piv, L.i32p)))
        self._top = (np.asfortranarray(lu), piv)

    @property
    def top_lu(self):
        if self._top is None:
            self._fetch_top()
        return self._top[0]

    @property
    def top_piv(self):
        if self._top is None:
            self._fetch_top()
        return self._top[1]

    @property
    def handle(self):
        return self._h

    def nbytes(self):
        return self._nbytes

    def max_rank(self):
        return max((rec.max_rank for rec in self.records), default=0)


def factorize(h2, eps_lu, threads=1, norm_estimate=None):
    """Factor a hierarchical matrix for fast solves (factorization.py:204-271).

    The input must have orthonormal bases; its blocks are not modified.
    Raises FactorizationError when a redundant diagonal block is singular.
    """
    del threads  # API parity: clusters of a batch run as one device launch
    return factorize_with(h2, eps_lu, norm_estimate)


def factorize_with(h2, eps_lu, norm_estimate=None, comm=None):
    """factorize() through h2f_factorize, or -- with `comm` (an h2f_comm,
    see multigpu.TorchComm) -- through h2f_factorize_sharded."""
    dev = device_matrix(h2)
    v0 = None
    if norm_estimate is None:
        v0 = np.ascontiguousarray(power_start(dev.n))
        est = -1.0
    else:
        est = float(norm_estimate)
    handle = C.c_void_p()
    st = L.Status()
    v0p = L.ptr(v0) if v0 is not None else None
    if comm is None:
        code = L.lib().h2f_factorize(dev.handle, float(eps_lu), est, v0p, C.byref(handle), C.byref(st))
    else:
        code = L.lib().h2f_factorize_sharded(dev.handle, float(eps_lu), est, v0p, C.byref(comm.struct),
                                             C.byref(handle), C.byref(st))
        comm.reraise()
    if code == L.H2F_E_SINGULAR:
        raise FactorizationError(L.last_error())
    L.check(code, "h2f_factorize" if comm is None else "h2f_factorize_sharded")
    return H2Factorization(h2.tree, _Handle(handle, dev))
