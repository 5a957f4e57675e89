"""Device construction of the H2 input.

`build_h2` + `orthogonalize_recompress` (/root/reference/pkg/src/h2factor/
h2core.py:128-269) run on the B200 through `h2f_matrix_build`
(include/h2f.h; csrc/build.cpp, csrc/k_build.cu): Chebyshev grids, Lagrange
leaf bases and transfers, kernel-evaluated couplings and dense near-field
blocks, then the QR / SVD-truncation / QR recompression sweeps -- the
operator never exists on the host.  The point set, the cluster tree and the
block partition (integer work, problem.py) stay host-side.

The result is a `DeviceH2`: the fields factorize / solve / matvec read
(tree, partition, rank, n) plus the device handle; its blocks can be exported
to host dicts on demand (`.leaf_basis` etc.), e.g. for the reference's own
code.  Tolerance contract (not bit-exact): GPU transcendental
functions and batched QR/SVD round differently from NumPy/LAPACK, and the
recompression projects a level's couplings after all of the level's SVDs
(csrc/build.cpp header).
"""
from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib as L
from . import problem as P
from .h2core import as_i64

__all__ = ["DeviceH2", "build_h2_device", "build_problem_device", "absorb_low_rank_device", "FAMILY_CODES"]

FAMILY_CODES = {"exp_covariance": 0, "laplace2d": 1, "helmholtz3d": 2}


class _BuiltMatrix:
    """h2f_matrix handle of a device-built operator (what device_matrix returns)."""

    def __init__(self, handle, n, nbytes):
        self.handle = handle
        self.n = n
        self.nbytes = nbytes
        self.key = None

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and L._lib is not None:
            L._lib.h2f_matrix_destroy(h)
            self.handle = None


class DeviceH2:
    """H2 operator built and resident on the device.  Same fields as the
    reference H2Matrix (h2core.py:97-125); the block dicts are exported from
    the device the first time they are read."""

    def __init__(self, tree, partition, rank, built, seconds):
        self.tree = tree
        self.partition = partition
        self.rank = rank
        self._h2f_built = built
        self.build_seconds = seconds
        self._host = None

    @property
    def n(self):
        return self.tree.n

    def _export(self):
        if self._host is None:
            self._host = export_blocks(self)
        return self._host

    leaf_basis = property(lambda self: self._export()["leaf_basis"])
    transfer = property(lambda self: self._export()["transfer"])
    coupling = property(lambda self: self._export()["coupling"])
    dense = property(lambda self: self._export()["dense"])


def _pair_lists(pairs_by_level, nlev):
    flat, ptr = [], [0]
    for lv in range(nlev):
        for s, t in sorted(pairs_by_level[lv]) if lv < len(pairs_by_level) else []:
            flat += [int(s), int(t)]
        ptr.append(len(flat) // 2)
    return as_i64(flat), as_i64(ptr)


def _structure(tree, part):
    nlev = int(tree.depth) + 1
    adm, adm_ptr = _pair_lists(part.admissible_leaves, nlev)
    inner, inner_ptr = _pair_lists(part.inadmissible_inner, nlev)
    dense, dense_ptr = _pair_lists(part.inadmissible_leaves, nlev)
    return dict(parent=as_i64(tree.parent), left=as_i64(tree.child_left), right=as_i64(tree.child_right),
                level=as_i64(tree.level), begin=as_i64(tree.begin), end=as_i64(tree.end), adm=adm,
                adm_ptr=adm_ptr, inner=inner, inner_ptr=inner_ptr, dense=dense, dense_ptr=dense_ptr)


def build_h2_device(tree, partition, spec, p0, eps):
    """build_h2(tree, partition, spec, p0) followed by
    orthogonalize_recompress(h2, eps), on the device (eps <= 0: no
    recompression).  Returns a DeviceH2."""
    if spec.family not in FAMILY_CODES:
        raise ValueError(f"unknown kernel family {spec.family!r}")
    lib = L.ensure_init()
    st = _structure(tree, partition)
    pts = np.ascontiguousarray(tree.points, dtype=np.float64)
    lo = np.ascontiguousarray(tree.box_lo, dtype=np.float64)
    hi = np.ascontiguousarray(tree.box_hi, dtype=np.float64)
    top = partition.top_level
    d = L.BuildDesc(
        n=int(tree.n), dim=int(pts.shape[1]), depth=int(tree.depth), top_level=-1 if top is None else int(top),
        p0=int(p0), num_nodes=int(len(tree.parent)),
        parent=L.ptr(st["parent"], L.i64p), child_left=L.ptr(st["left"], L.i64p),
        child_right=L.ptr(st["right"], L.i64p), level=L.ptr(st["level"], L.i64p),
        begin=L.ptr(st["begin"], L.i64p), end=L.ptr(st["end"], L.i64p),
        points=L.ptr(pts), box_lo=L.ptr(lo), box_hi=L.ptr(hi),
        adm_pairs=L.ptr(st["adm"], L.i64p), adm_ptr=L.ptr(st["adm_ptr"], L.i64p),
        inner_pairs=L.ptr(st["inner"], L.i64p), inner_ptr=L.ptr(st["inner_ptr"], L.i64p),
        dense_pairs=L.ptr(st["dense"], L.i64p), dense_ptr=L.ptr(st["dense_ptr"], L.i64p),
        family=FAMILY_CODES[spec.family], corr_length=float(spec.corr_length), kappa=float(spec.kappa),
        diag_value=float(spec.diag_value), alpha_r=float(spec.alpha_r), eps=float(eps))
    handle = C.c_void_p()
    rank = np.empty(len(tree.parent), dtype=np.int64)
    secs = np.zeros(2)
    L.check(lib.h2f_matrix_build(C.byref(d), C.byref(handle), L.ptr(rank, L.i64p), L.ptr(secs)),
            "h2f_matrix_build")
    nb = C.c_int64()
    L.check(lib.h2f_matrix_nbytes(handle, C.byref(nb)), "h2f_matrix_nbytes")
    built = _BuiltMatrix(handle, int(tree.n), int(nb.value))
    ranks = {int(c): int(k) for c, k in enumerate(rank) if k >= 0}
    h2 = DeviceH2(tree, partition, ranks, built,
                  {"construction": float(secs[0]), "compression": float(secs[1])})
    h2._st = st
    return h2


def absorb_low_rank_device(h2, w, eps):
    """absorb_low_rank(h2, w, eps) (h2core.py:342-405) on the device: a new
    DeviceH2 for A + W W^T, recompressed at eps.  h2 (host H2Matrix or
    DeviceH2) is not modified -- unlike the reference, which updates in
    place, the device operator is immutable.  W: n x r in tree order."""
    from .h2core import device_matrix

    w = np.ascontiguousarray(np.asarray(w, dtype=np.float64))
    if w.ndim != 2 or w.shape[0] != h2.n:
        raise ValueError("update factor must be n x r")
    lib = L.ensure_init()
    src = device_matrix(h2)
    handle = C.c_void_p()
    rank = np.empty(len(h2.tree.parent), dtype=np.int64)
    secs = np.zeros(2)
    L.check(lib.h2f_matrix_absorb_low_rank(src.handle, L.ptr(w), int(w.shape[1]), float(eps), C.byref(handle),
                                           L.ptr(rank, L.i64p), L.ptr(secs)), "h2f_matrix_absorb_low_rank")
    nb = C.c_int64()
    L.check(lib.h2f_matrix_nbytes(handle, C.byref(nb)), "h2f_matrix_nbytes")
    built = _BuiltMatrix(handle, int(h2.n), int(nb.value))
    ranks = {int(c): int(k) for c, k in enumerate(rank) if k >= 0}
    out = DeviceH2(h2.tree, h2.partition, ranks, built,
                   {"low_rank_update": float(secs[0]), "compression": float(secs[1])})
    out._st = getattr(h2, "_st", None) or _structure(h2.tree, h2.partition)
    return out


def export_blocks(h2):
    """The device operator's blocks as the reference's dicts (one D2H copy)."""
    lib = L.lib()
    st = h2._st
    nn = len(h2.tree.parent)
    na, nd = int(st["adm_ptr"][-1]), int(st["dense_ptr"][-1])
    lo, to = np.empty(nn, np.int64), np.empty(nn, np.int64)
    co, do = np.empty(max(na, 1), np.int64), np.empty(max(nd, 1), np.int64)
    nv = C.c_int64()
    h = h2._h2f_built.handle
    L.check(lib.h2f_matrix_layout(h, L.ptr(lo, L.i64p), L.ptr(to, L.i64p), L.ptr(co, L.i64p),
                                  L.ptr(do, L.i64p), C.byref(nv)), "h2f_matrix_layout")
    vals = np.empty(max(nv.value, 1))
    L.check(lib.h2f_matrix_values(h, L.ptr(vals)), "h2f_matrix_values")
    tree, rank = h2.tree, h2.rank
    out = {"leaf_basis": {}, "transfer": {}, "coupling": {}, "dense": {}}
    for c in range(nn):
        if lo[c] >= 0:
            m, k = tree.size(c), rank[c]
            out["leaf_basis"][c] = vals[lo[c]:lo[c] + m * k].reshape(m, k).copy()
        if to[c] >= 0:
            k, kp = rank[c], rank[int(tree.parent[c])]
            out["transfer"][c] = vals[to[c]:to[c] + k * kp].reshape(k, kp).copy()
    adm = st["adm"].reshape(-1, 2)
    for i in range(na):
        s, t = int(adm[i, 0]), int(adm[i, 1])
        ks, kt = rank[s], rank[t]
        out["coupling"][(s, t)] = vals[co[i]:co[i] + ks * kt].reshape(ks, kt).copy()
    dense = st["dense"].reshape(-1, 2)
    for i in range(nd):
        s, t = int(dense[i, 0]), int(dense[i, 1])
        ms, mt = tree.size(s), tree.size(t)
        out["dense"][(s, t)] = vals[do[i]:do[i] + ms * mt].reshape(ms, mt).copy()
    return out


def build_problem_device(name, n, **overrides):
    """problem.build_problem with the operator built on the device:
    (tree, partition, spec, DeviceH2, params).  The low-rank-update row
    (lru_rank > 0) is not supported here."""
    if name not in P.PROBLEMS:
        raise ValueError(f"unknown problem {name!r}; choose from {sorted(P.PROBLEMS)}")
    prm = dict(P.PROBLEMS[name])
    prm.update({k: v for k, v in overrides.items() if v is not None})
    t0 = time.perf_counter()
    points, counts = P.generate_uniform_grid(n, prm["dim"])
    h = 1.0 / max(counts)
    tree = P.build_cluster_tree(points, prm["m"])
    part = P.dual_tree_traversal(tree, prm["eta"])
    spec = P.KernelSpec(family=prm["family"], dim=prm["dim"], corr_length=prm["corr_length"],
                        kappa=prm["kappa"], diag_value=P.default_diag_value(prm["family"], h),
                        alpha_r=prm["alpha_r"])
    t1 = time.perf_counter()
    h2 = build_h2_device(tree, part, spec, prm["p0"], prm["eps"])
    h2.build_seconds["host_structure"] = t1 - t0
    if prm.get("lru_rank", 0) > 0:
        # the low-rank row (harness.py:68-70, 185-189): seeded W, absorbed on the device
        # (rows in tree order, as problem._build passes it to absorb_low_rank)
        w = P.make_low_rank_factor(n, prm["lru_rank"], prm.get("seed", 7))
        h2u = absorb_low_rank_device(h2, w, prm["eps"])
        h2u.build_seconds = dict(h2.build_seconds, **{"low_rank_update": h2u.build_seconds["low_rank_update"],
                                                       "compression_after_update": h2u.build_seconds["compression"]})
        h2 = h2u
    h2.build_seconds["device_total"] = time.perf_counter() - t1
    return tree, part, spec, h2, prm
