"""Device-resident H2 operator, matvec and the norm estimate.

Mirrors h2core.matvec / estimate_norm2 (/root/reference/pkg/src/h2factor/
h2core.py:285-330).  Any object with the reference H2Matrix fields (tree,
partition, leaf_basis, transfer, coupling, dense, rank) is accepted, so both
the reference's H2Matrix and paper_2509_11152_b200.problem.H2Matrix work.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L

__all__ = ["DeviceMatrix", "device_matrix", "matvec", "estimate_norm2", "power_start"]


def _fingerprint(h2):
    # block replacement (e.g. h2.dense[key] = new array) invalidates the
    # upload; blocks are treated as immutable in place, like the reference
    # (factorization.py:207-208 "its blocks are not modified")
    ids = []
    for store in (h2.leaf_basis, h2.transfer, h2.coupling, h2.dense):
        ids.append(len(store))
        ids.extend(id(v) for v in store.values())
    return hash(tuple(ids)), id(h2.tree), id(h2.partition)


class DeviceMatrix:
    """An H2 operator uploaded to the B200 (h2f_matrix)."""

    def __init__(self, h2):
        tree, part = h2.tree, h2.partition
        n = int(tree.n)
        nnodes = int(len(tree.parent))
        depth = int(tree.depth)
        nlev = depth + 1
        top = part.top_level
        rank = np.full(nnodes, -1, dtype=np.int64)
        for c, k in h2.rank.items():
            rank[int(c)] = int(k)
        blocks = []  # (flat block, offset in the value array)
        pos = 0

        def place(arr):
            nonlocal pos
            a = np.ascontiguousarray(arr, dtype=np.float64)
            blocks.append((a.ravel(), pos))
            off = pos
            pos += a.size
            return off

        leaf_off = np.full(nnodes, -1, dtype=np.int64)
        for c, blk in h2.leaf_basis.items():
            leaf_off[int(c)] = place(blk)
        trans_off = np.full(nnodes, -1, dtype=np.int64)
        for c, blk in h2.transfer.items():
            trans_off[int(c)] = place(blk)

        def level_lists(pairs_by_level, store):
            flat, ptr, offs = [], [0], []
            for lv in range(nlev):
                pairs = sorted(pairs_by_level[lv]) if lv < len(pairs_by_level) else []
                for s, t in pairs:
                    flat += [int(s), int(t)]
                    if store is not None:
                        offs.append(place(store[(s, t)]))
                ptr.append(len(flat) // 2)
            return as_i64(flat), as_i64(ptr), as_i64(offs)

        adm = [list(p) for p in part.admissible_leaves]
        inner = [list(p) for p in part.inadmissible_inner]
        dense_lv = [[] for _ in range(nlev)]
        for (s, t) in h2.dense:
            dense_lv[int(tree.level[s])].append((int(s), int(t)))
        adm_pairs, adm_ptr, coup_off = level_lists(adm, h2.coupling)
        inner_pairs, inner_ptr, _ = level_lists(inner, None)
        dense_pairs, dense_ptr, dense_off = level_lists(dense_lv, h2.dense)
        nvals = max(pos, 1)
        keep = dict(parent=as_i64(tree.parent), left=as_i64(tree.child_left),
                    right=as_i64(tree.child_right), level=as_i64(tree.level),
                    begin=as_i64(tree.begin), end=as_i64(tree.end), rank=rank,
                    adm_pairs=adm_pairs, adm_ptr=adm_ptr, inner_pairs=inner_pairs,
                    inner_ptr=inner_ptr, dense_pairs=dense_pairs, dense_ptr=dense_ptr,
                    leaf_off=leaf_off, trans_off=trans_off, coup_off=coup_off, dense_off=dense_off)
        p = {k: L.ptr(v, L.i64p) for k, v in keep.items()}
        desc = L.MatrixDesc(
            n=n, depth=depth, top_level=-1 if top is None else int(top), num_nodes=nnodes,
            parent=p["parent"], child_left=p["left"], child_right=p["right"], level=p["level"],
            begin=p["begin"], end=p["end"], rank=p["rank"],
            adm_pairs=p["adm_pairs"], adm_ptr=p["adm_ptr"], inner_pairs=p["inner_pairs"],
            inner_ptr=p["inner_ptr"], dense_pairs=p["dense_pairs"], dense_ptr=p["dense_ptr"],
            leaf_basis_off=p["leaf_off"], transfer_off=p["trans_off"], coupling_off=p["coup_off"],
            dense_off=p["dense_off"], nvals=int(nvals))
        lib = L.ensure_init()
        handle = C.c_void_p()
        # the blocks as they are (no packed host copy): the library packs
        # pinned chunks in parallel, overlapped with the upload
        nb = len(blocks)
        ptrs = (C.c_void_p * max(nb, 1))(*[a.ctypes.data for a, _ in blocks])
        counts = np.fromiter((a.size for a, _ in blocks), dtype=np.int64, count=nb)
        offs = np.fromiter((o for _, o in blocks), dtype=np.int64, count=nb)
        L.check(lib.h2f_matrix_create_blocks(C.byref(desc), nb, ptrs, L.ptr(counts, L.i64p), L.ptr(offs, L.i64p),
                                             C.byref(handle)), "h2f_matrix_create_blocks")
        del blocks
        self.handle = handle
        self.n = n
        self.nbytes = int(nvals) * 8
        self.key = _fingerprint(h2)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and L._lib is not None:
            L._lib.h2f_matrix_destroy(h)
            self.handle = None


def as_i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64).reshape(-1))


def device_matrix(h2):
    """Upload h2 once and cache the handle on the object (a DeviceH2 from
    construct.py already lives on the device)."""
    built = getattr(h2, "_h2f_built", None)
    if built is not None:
        return built
    dev = getattr(h2, "_h2f_device", None)
    if dev is not None and dev.key == _fingerprint(h2):
        return dev
    dev = DeviceMatrix(h2)
    try:
        object.__setattr__(h2, "_h2f_device", dev)
    except (AttributeError, TypeError):
        pass
    return dev


def matvec(h2, x):
    """y = A x in tree order (h2core.py:285-315); x may be (n,) or (n, q)."""
    x = np.asarray(x, dtype=np.float64)
    dev = device_matrix(h2)
    if x.shape[0] != dev.n or x.ndim not in (1, 2):
        raise ValueError(f"vector must have shape ({dev.n},) or ({dev.n}, q)")
    xc = np.ascontiguousarray(x)
    y = np.empty_like(xc)
    nrhs = 1 if x.ndim == 1 else x.shape[1]
    L.check(L.lib().h2f_matvec(dev.handle, L.ptr(xc), L.ptr(y), nrhs), "h2f_matvec")
    return y


def power_start(n, seed=20240901):
    """Normalised Philox start vector of estimate_norm2 (h2core.py:320-322)."""
    v = np.random.Generator(np.random.Philox(seed)).standard_normal(n)
    return v / np.linalg.norm(v)


def estimate_norm2(h2, iters=30, seed=20240901):
    """Spectral-norm estimate by power iteration (h2core.py:318-330)."""
    dev = device_matrix(h2)
    v = np.ascontiguousarray(power_start(dev.n, seed))
    est = C.c_double()
    L.check(L.lib().h2f_norm2(dev.handle, L.ptr(v), int(iters), C.byref(est)), "h2f_norm2")
    return float(est.value)
