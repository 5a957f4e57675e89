"""ctypes binding of libh2f.so (include/h2f.h).

The library is required: there is no CPU fallback anywhere in the package.
Importing works without a GPU (so the CPU test suite can check the exported
symbols); the first compute call initialises the CUDA context and raises if
no device or no library is available.
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("H2F_LIB", os.path.join(HERE, "libh2f.so"))  # H2F_LIB: development builds
HEADER = os.path.join(os.path.dirname(HERE), "include", "h2f.h")

H2F_OK, H2F_E_ARG, H2F_E_CUDA, H2F_E_NOMEM, H2F_E_SINGULAR, H2F_E_INTERNAL = range(6)

i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)


class MatrixDesc(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("depth", C.c_int32), ("top_level", C.c_int32), ("num_nodes", C.c_int64),
        ("parent", i64p), ("child_left", i64p), ("child_right", i64p), ("level", i64p),
        ("begin", i64p), ("end", i64p), ("rank", i64p),
        ("adm_pairs", i64p), ("adm_ptr", i64p),
        ("inner_pairs", i64p), ("inner_ptr", i64p),
        ("dense_pairs", i64p), ("dense_ptr", i64p),
        ("leaf_basis_off", i64p), ("transfer_off", i64p), ("coupling_off", i64p), ("dense_off", i64p),
        ("nvals", C.c_int64),
    ]


class BuildDesc(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("dim", C.c_int32), ("depth", C.c_int32), ("top_level", C.c_int32),
        ("p0", C.c_int32), ("num_nodes", C.c_int64),
        ("parent", i64p), ("child_left", i64p), ("child_right", i64p), ("level", i64p),
        ("begin", i64p), ("end", i64p),
        ("points", f64p), ("box_lo", f64p), ("box_hi", f64p),
        ("adm_pairs", i64p), ("adm_ptr", i64p),
        ("inner_pairs", i64p), ("inner_ptr", i64p),
        ("dense_pairs", i64p), ("dense_ptr", i64p),
        ("family", C.c_int32), ("pad_", C.c_int32),
        ("corr_length", C.c_double), ("kappa", C.c_double), ("diag_value", C.c_double),
        ("alpha_r", C.c_double), ("eps", C.c_double),
    ]


class KernelProfile(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("seconds", C.c_double),
                ("flops", C.c_double), ("bytes", C.c_double)]


class Status(C.Structure):
    _fields_ = [("code", C.c_int32), ("cluster", C.c_int32), ("level", C.c_int32)]


class FactorInfo(C.Structure):
    _fields_ = [("n", C.c_int64), ("top_level", C.c_int32), ("num_records", C.c_int32),
                ("top_size", C.c_int64), ("eps_lu", C.c_double), ("eps_fill", C.c_double),
                ("norm_estimate", C.c_double), ("nbytes", C.c_int64),
                ("phase_seconds", C.c_double * 8)]


class LevelInfo(C.Structure):
    _fields_ = [("level", C.c_int32), ("num_clusters", C.c_int32), ("num_batches", C.c_int32),
                ("csp", C.c_int32), ("ncolors", C.c_int32), ("graph_degree", C.c_int32),
                ("max_rank", C.c_int32), ("total_size", C.c_int64), ("up_size", C.c_int64),
                ("batch_entries", C.c_int64), ("time_s", C.c_double)]


class ClusterInfo(C.Structure):
    _fields_ = [("cluster", C.c_int32), ("level", C.c_int32), ("size", C.c_int32), ("r", C.c_int32),
                ("num_edges", C.c_int32), ("offset", C.c_int64)]


# collective callbacks of h2f_comm (include/h2f.h)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, f64p, C.c_int64)
ALLREDUCE_DEV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64)
ALLTOALLV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, i64p, C.c_void_p, i64p)
BROADCAST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32)


class Comm(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("user", C.c_void_p),
                ("allreduce_max", ALLREDUCE_FN), ("allreduce_sum_dev", ALLREDUCE_DEV_FN),
                ("alltoallv_dev", ALLTOALLV_FN), ("broadcast_dev", BROADCAST_FN)]


_SIGS = {
    "h2f_init": (C.c_int, [C.c_int, C.c_double]),
    "h2f_last_error": (C.c_char_p, []),
    "h2f_stream": (C.c_int, [C.POINTER(C.c_void_p)]),
    "h2f_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "h2f_kernel_launches": (C.c_int, [i64p]),
    "h2f_memory_stats": (C.c_int, [i64p, i64p, i64p]),
    "h2f_profile_enable": (C.c_int, [C.c_int]),
    "h2f_profile_reset": (C.c_int, []),
    "h2f_profile_count": (C.c_int, [i32p]),
    "h2f_profile_get": (C.c_int, [C.c_int32, C.POINTER(KernelProfile)]),
    "h2f_bench_dmma": (C.c_int, [C.c_int64, f64p]),
    "h2f_dense_svd": (C.c_int, [f64p, C.c_int32, C.c_int32, C.c_double, C.c_int32, f64p, i32p, i32p, f64p]),
    "h2f_dense_qr_r": (C.c_int, [f64p, C.c_int32, C.c_int32, C.c_int32, f64p, f64p]),
    "h2f_dense_complement": (C.c_int, [f64p, C.c_int32, C.c_int32, C.c_int32, f64p, f64p]),
    "h2f_matrix_create": (C.c_int, [C.POINTER(MatrixDesc), f64p, C.POINTER(C.c_void_p)]),
    "h2f_matrix_create_blocks": (C.c_int, [C.POINTER(MatrixDesc), C.c_int64, C.POINTER(C.c_void_p), i64p, i64p,
                                           C.POINTER(C.c_void_p)]),
    "h2f_matrix_destroy": (C.c_int, [C.c_void_p]),
    "h2f_matrix_nbytes": (C.c_int, [C.c_void_p, i64p]),
    "h2f_matrix_build": (C.c_int, [C.POINTER(BuildDesc), C.POINTER(C.c_void_p), i64p, f64p]),
    "h2f_matrix_absorb_low_rank": (C.c_int, [C.c_void_p, f64p, C.c_int32, C.c_double, C.POINTER(C.c_void_p),
                                             i64p, f64p]),
    "h2f_matrix_layout": (C.c_int, [C.c_void_p, i64p, i64p, i64p, i64p, i64p]),
    "h2f_matrix_values": (C.c_int, [C.c_void_p, f64p]),
    "h2f_matvec": (C.c_int, [C.c_void_p, f64p, f64p, C.c_int64]),
    "h2f_matvec_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]),
    "h2f_norm2": (C.c_int, [C.c_void_p, f64p, C.c_int32, f64p]),
    "h2f_factorize": (C.c_int, [C.c_void_p, C.c_double, C.c_double, f64p, C.POINTER(C.c_void_p),
                                C.POINTER(Status)]),
    "h2f_factorize_sharded": (C.c_int, [C.c_void_p, C.c_double, C.c_double, f64p, C.POINTER(Comm),
                                        C.POINTER(C.c_void_p), C.POINTER(Status)]),
    "h2f_shard_stats": (C.c_int, [f64p]),
    "h2f_shard_owners": (C.c_int, [C.c_int64, i64p, i64p, C.c_int32, C.c_int32, i32p]),
    "h2f_factor_destroy": (C.c_int, [C.c_void_p]),
    "h2f_solve": (C.c_int, [C.c_void_p, f64p, f64p, C.c_int64]),
    "h2f_solve_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]),
    "h2f_refined_solve": (C.c_int, [C.c_void_p, C.c_void_p, f64p, f64p, C.c_int32]),
    "h2f_refined_solve_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32]),
    "h2f_refined_solve_multi": (C.c_int, [C.c_void_p, C.c_void_p, f64p, f64p, C.c_int64, C.c_int32]),
    "h2f_refined_solve_multi_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                              C.c_int32]),
    "h2f_factor_import_begin": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.c_int64, C.c_double, C.c_double,
                                          C.c_double, C.POINTER(C.c_void_p)]),
    "h2f_factor_import_record": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, i64p, i64p, i64p, C.c_int32,
                                           i64p, i64p, C.c_int64, i64p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                           C.c_double]),
    "h2f_factor_import_cluster": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, f64p, f64p,
                                            i32p, C.c_int32, i64p, i32p, i64p, f64p]),
    "h2f_factor_import_top": (C.c_int, [C.c_void_p, f64p, i32p]),
    "h2f_factor_import_end": (C.c_int, [C.c_void_p]),
    "h2f_factor_info_get": (C.c_int, [C.c_void_p, C.POINTER(FactorInfo)]),
    "h2f_factor_level_info": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(LevelInfo)]),
    "h2f_factor_level_arrays": (C.c_int, [C.c_void_p, C.c_int32, i64p, i64p, i64p, i64p, i64p, i64p]),
    "h2f_factor_level_fills": (C.c_int, [C.c_void_p, C.c_int32, i64p, i64p, i64p, i64p]),
    "h2f_factor_cluster_info": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(ClusterInfo)]),
    "h2f_factor_cluster_arrays": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, f64p, f64p, i32p, i64p,
                                            i32p, i64p]),
    "h2f_factor_cluster_edge": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, f64p]),
    "h2f_factor_top": (C.c_int, [C.c_void_p, f64p, i32p]),
    "h2f_greedy_coloring": (C.c_int, [C.c_int64, i64p, C.c_int64, i64p, i32p, i32p, i32p]),
    "h2f_debug_replay_set": (C.c_int, [i64p, C.c_int64, i64p, C.c_int64]),
    "h2f_debug_replay_clear": (C.c_int, []),
    "h2f_debug_replay_stats": (C.c_int, [i64p]),
}

_lib = None
_initialised = False
_device = None


class H2FError(RuntimeError):
    """A failure reported by libh2f (CUDA error, arena exhausted, ...)."""


def header_symbols():
    """Function names declared in include/h2f.h."""
    with open(HEADER) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(h2f_[a-z0-9_]+)\s*\(", text)))


def lib():
    """The loaded library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2509_11152_b200.build` "
                              "(there is no CPU fallback)")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def last_error():
    msg = lib().h2f_last_error()
    return msg.decode() if msg else ""


def check(code, what=""):
    if code == H2F_OK:
        return
    msg = last_error()
    if code == H2F_E_ARG:
        raise ValueError(msg)
    if code == H2F_E_INTERNAL:
        raise AssertionError(msg)
    raise H2FError(f"{what}: {msg}" if what else msg)


def ensure_init(device=None):
    """Create the library's CUDA context (once per process).

    Device: the argument, else H2F_DEVICE, else LOCAL_RANK (one process per
    GPU under torchrun), else 0."""
    global _initialised, _device
    if not _initialised:
        if device is None:
            device = int(os.environ.get("H2F_DEVICE", os.environ.get("LOCAL_RANK", "0")))
        dev = int(device)
        arena = float(os.environ.get("H2F_ARENA_GB", "0"))
        check(lib().h2f_init(dev, arena), "h2f_init")
        _initialised = True
        _device = dev
    return lib()


def device():
    """CUDA ordinal the library context lives on (initialises it)."""
    ensure_init()
    return _device


def ptr(a, typ=f64p):
    return a.ctypes.data_as(typ)


def as_f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def as_i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def kernel_launches():
    v = C.c_int64()
    lib().h2f_kernel_launches(C.byref(v))
    return v.value


def stream_handle():
    s = C.c_void_p()
    check(ensure_init().h2f_stream(C.byref(s)))
    return s.value


def memory_stats():
    a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
    check(ensure_init().h2f_memory_stats(C.byref(a), C.byref(b), C.byref(c)))
    return {"arena_bytes": a.value, "in_use": b.value, "peak": c.value}


def profile_enable(on=True):
    check(ensure_init().h2f_profile_enable(1 if on else 0))


def profile_reset():
    check(ensure_init().h2f_profile_reset())


def profile_get():
    """{kernel name: {launches, seconds, flops, bytes}} since the last reset."""
    n = C.c_int32()
    check(lib().h2f_profile_count(C.byref(n)))
    out = {}
    for k in range(n.value):
        p = KernelProfile()
        check(lib().h2f_profile_get(k, C.byref(p)))
        if p.launches:
            out[p.name.decode()] = {"launches": p.launches, "seconds": p.seconds, "flops": p.flops,
                                    "bytes": p.bytes}
    return out


def bench_dmma(iters=20000):
    v = C.c_double()
    check(ensure_init().h2f_bench_dmma(int(iters), C.byref(v)))
    return v.value


# ---- per-cluster dense kernels (test / micro-benchmark hooks) ---------------

def dense_svd(R, thresh, path):
    """(U_kept, kept, sweeps, ms): one-sided Jacobi on the rows of R (m x n)."""
    R = as_f64(R)
    m, n = R.shape
    U = np.zeros((n, n))
    kept, sweeps, ms = C.c_int32(), C.c_int32(), C.c_double()
    check(ensure_init().h2f_dense_svd(ptr(R), m, n, float(thresh), int(path), ptr(U), C.byref(kept),
                                      C.byref(sweeps), C.byref(ms)))
    return U[:kept.value].copy(), kept.value, sweeps.value, ms.value


def dense_qr_r(Y, path):
    """(R, ms): R factor of the QR of Y^T (Y is n x wf)."""
    Y = as_f64(Y)
    n, wf = Y.shape
    R = np.zeros((min(n, wf), n))
    ms = C.c_double()
    check(ensure_init().h2f_dense_qr_r(ptr(Y), n, wf, int(path), ptr(R), C.byref(ms)))
    return R, ms.value


def dense_complement(BT, path):
    """(Q, ms): [orthonormal complement | b_aug] from BT = b_aug^T (kt x s)."""
    BT = as_f64(BT)
    kt, s = BT.shape
    Q = np.zeros((s, s))
    ms = C.c_double()
    check(ensure_init().h2f_dense_complement(ptr(BT), s, kt, int(path), ptr(Q), C.byref(ms)))
    return Q, ms.value


# ---- structure replay (parity diagnostics) ----------------------------------

def replay_set(kept_rows, created_rows):
    """Force the threshold decisions of another run: kept_rows (k, 3) =
    (level, cluster, kept), created_rows (f, 4) = (level, creator, a, b)."""
    k = as_i64(np.asarray(kept_rows).reshape(-1, 3))
    f = as_i64(np.asarray(created_rows).reshape(-1, 4))
    check(ensure_init().h2f_debug_replay_set(ptr(k, i64p), k.shape[0], ptr(f, i64p), f.shape[0]))


def replay_clear():
    check(ensure_init().h2f_debug_replay_clear())


def replay_stats():
    st = np.zeros(8, dtype=np.int64)
    check(ensure_init().h2f_debug_replay_stats(ptr(st, i64p)))
    return {"kept_forced": int(st[0]), "kept_changed": int(st[1]), "fill_changed": int(st[2]),
            "fill_changed_by_log10_margin": {"<0.01": int(st[3]), "<0.1": int(st[4]), "<0.5": int(st[5]),
                                             "<1": int(st[6]), ">=1": int(st[7])}}
