"""On-disk / wire format of a B200 factorization.

The reference has no serialization (its H2Factorization is an in-memory
object, /root/reference/pkg/src/h2factor/factorization.py:167-193).  A
factor here lives in device memory; `save_factorization` exports every
field the solve needs (records, per-cluster q / lu / piv / eliminator
edges, the dense top LU) into one .npz, `load_factorization` rebuilds the
device factor through the import half of the C ABI (h2f_factor_import_*).
The loaded factor solves bit-for-bit like the saved one.  `pack` / `unpack`
give the same content as a dict of NumPy arrays, which multigpu.py
broadcasts to reuse one factorization on every rank (config 5) instead of
re-factoring.

Format "h2f-factor-1": meta (JSON), top_lu / top_piv, and per record r
rec{r}_{clusters,offsets,sizes,batch_ptr,batch_ids,up_index,attrs} plus the
clusters' arrays concatenated in record order with offset vectors
(q, lu, piv, edge other/kind/width, mw = r x sum(widths) per cluster).
"""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from . import _lib as L
from .factorization import H2Factorization, _Handle

__all__ = ["save_factorization", "load_factorization", "pack", "unpack"]

FORMAT = "h2f-factor-1"
_KIND_CODE = {"self": 0, "full": 1, "skel": 2}


def pack(fac):
    """Dict of arrays holding the whole factor (host copies)."""
    out = {}
    meta = {"format": FORMAT, "n": fac.n, "top_level": -1 if fac.top_level is None else fac.top_level,
            "records": len(fac.records), "top_size": fac.top_size, "eps_lu": fac.eps_lu,
            "eps_fill": fac.eps_fill, "norm_estimate": fac.norm_estimate, "nbytes": fac.nbytes(),
            "phase_seconds": fac.phase_seconds}
    out["meta"] = np.array(json.dumps(meta))
    out["top_lu"] = np.ascontiguousarray(fac.top_lu) if fac.top_size else np.zeros(0)
    out["top_piv"] = np.ascontiguousarray(fac.top_piv, dtype=np.int32) if fac.top_size else np.zeros(0, np.int32)
    for i, rec in enumerate(fac.records):
        p = f"rec{i}_"
        out[p + "clusters"] = np.array(rec.clusters, dtype=np.int64)
        out[p + "offsets"] = np.array([rec.offset[c] for c in rec.clusters], dtype=np.int64)
        out[p + "sizes"] = np.array([rec.size[c] for c in rec.clusters], dtype=np.int64)
        out[p + "batch_ptr"] = np.cumsum([0] + [len(b) for b in rec.batches]).astype(np.int64)
        out[p + "batch_ids"] = np.array([c for b in rec.batches for c in b], dtype=np.int64)
        out[p + "up_index"] = np.asarray(rec.up_index, dtype=np.int64)
        out[p + "attrs"] = np.array([rec.level, rec.csp, rec.ncolors, rec.graph_degree, rec.max_rank], np.int64)
        out[p + "time_s"] = np.array([rec.time_s])
        rs, qs, lus, pivs, ne, eo, ek, ew, mws = [], [], [], [], [], [], [], [], []
        for c in rec.clusters:
            f = rec.factors[c]
            rs.append(f.r)
            qs.append(np.ascontiguousarray(f.q).ravel())
            if f.r:
                lus.append(np.ascontiguousarray(f.lu).ravel())
                pivs.append(np.asarray(f.piv, dtype=np.int32))
                ne.append(len(f.edges))
                for o, k, m in f.edges:
                    eo.append(o)
                    ek.append(_KIND_CODE[k])
                    ew.append(m.shape[1])
                mws.append(np.hstack([m for _, _, m in f.edges]).ravel() if f.edges else np.zeros(0))
            else:
                ne.append(0)
        out[p + "r"] = np.array(rs, dtype=np.int64)
        out[p + "q"] = np.concatenate(qs) if qs else np.zeros(0)
        out[p + "lu"] = np.concatenate(lus) if lus else np.zeros(0)
        out[p + "piv"] = np.concatenate(pivs) if pivs else np.zeros(0, np.int32)
        out[p + "nedges"] = np.array(ne, dtype=np.int64)
        out[p + "edge_other"] = np.array(eo, dtype=np.int64)
        out[p + "edge_kind"] = np.array(ek, dtype=np.int32)
        out[p + "edge_width"] = np.array(ew, dtype=np.int64)
        out[p + "mw"] = np.concatenate(mws) if mws else np.zeros(0)
    return out


def unpack(arrays, tree=None):
    """Device factor from a dict produced by pack (or a loaded .npz)."""
    meta = json.loads(str(arrays["meta"]))
    if meta.get("format") != FORMAT:
        raise ValueError(f"not an {FORMAT} archive")
    lib = L.ensure_init()
    h = C.c_void_p()
    L.check(lib.h2f_factor_import_begin(int(meta["n"]), int(meta["top_level"]), int(meta["records"]),
                                        int(meta["top_size"]), float(meta["eps_lu"]), float(meta["eps_fill"]),
                                        float(meta["norm_estimate"]), C.byref(h)), "h2f_factor_import_begin")
    handle = _Handle(h, None)  # owns the factor from here on (freed on error)
    i64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)  # noqa: E731
    for i in range(int(meta["records"])):
        p = f"rec{i}_"
        cl, offs, sizes = i64(arrays[p + "clusters"]), i64(arrays[p + "offsets"]), i64(arrays[p + "sizes"])
        bptr, bids, up = i64(arrays[p + "batch_ptr"]), i64(arrays[p + "batch_ids"]), i64(arrays[p + "up_index"])
        lvl, csp, ncol, deg, mr = (int(v) for v in arrays[p + "attrs"])
        L.check(lib.h2f_factor_import_record(
            h, i, lvl, len(cl), L.ptr(cl, L.i64p), L.ptr(offs, L.i64p), L.ptr(sizes, L.i64p), len(bptr) - 1,
            L.ptr(bptr, L.i64p), L.ptr(bids if bids.size else np.zeros(1, np.int64), L.i64p), len(up),
            L.ptr(up if up.size else np.zeros(1, np.int64), L.i64p), csp, ncol, deg, mr,
            float(arrays[p + "time_s"][0])), "h2f_factor_import_record")
        rr, q, lu, piv = i64(arrays[p + "r"]), np.asarray(arrays[p + "q"]), np.asarray(arrays[p + "lu"]), \
            np.asarray(arrays[p + "piv"], dtype=np.int32)
        ne, eo = i64(arrays[p + "nedges"]), i64(arrays[p + "edge_other"])
        ek, ew = np.asarray(arrays[p + "edge_kind"], dtype=np.int32), i64(arrays[p + "edge_width"])
        mw = np.asarray(arrays[p + "mw"])
        qo = lo = po = eo_i = mo = 0
        for j, c in enumerate(cl):
            s, r = int(sizes[j]), int(rr[j])
            qc = np.ascontiguousarray(q[qo:qo + s * s])
            qo += s * s
            k = int(ne[j])
            if r:
                luc = np.ascontiguousarray(lu[lo:lo + r * r])
                pc = np.ascontiguousarray(piv[po:po + r])
                lo += r * r
                po += r
                oc, kc, wc = i64(eo[eo_i:eo_i + k]), np.ascontiguousarray(ek[eo_i:eo_i + k]), i64(ew[eo_i:eo_i + k])
                eo_i += k
                wsum = int(wc.sum())
                mc = np.ascontiguousarray(mw[mo:mo + r * wsum])
                mo += r * wsum
                L.check(lib.h2f_factor_import_cluster(h, i, int(c), s, r, L.ptr(qc), L.ptr(luc), L.ptr(pc, L.i32p),
                                                      k, L.ptr(oc, L.i64p), L.ptr(kc, L.i32p), L.ptr(wc, L.i64p),
                                                      L.ptr(mc)), "h2f_factor_import_cluster")
            else:
                L.check(lib.h2f_factor_import_cluster(h, i, int(c), s, 0, L.ptr(qc), None, None, 0, None, None,
                                                      None, None), "h2f_factor_import_cluster")
    if int(meta["top_size"]):
        tl = np.ascontiguousarray(arrays["top_lu"], dtype=np.float64)
        tp = np.ascontiguousarray(arrays["top_piv"], dtype=np.int32)
        L.check(lib.h2f_factor_import_top(h, L.ptr(tl), L.ptr(tp, L.i32p)), "h2f_factor_import_top")
    L.check(lib.h2f_factor_import_end(h), "h2f_factor_import_end")
    fac = H2Factorization(tree, handle)
    fac.phase_seconds = dict(meta.get("phase_seconds", {}))
    return fac


def save_factorization(fac, path):
    """Write the factor to `path` (.npz, uncompressed: FP64 factor data does
    not compress)."""
    np.savez(path, **pack(fac))


def load_factorization(path, tree=None):
    """Device factor from a file written by save_factorization."""
    with np.load(path, allow_pickle=False) as z:
        return unpack({k: z[k] for k in z.files}, tree)
