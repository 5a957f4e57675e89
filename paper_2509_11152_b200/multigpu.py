"""Multi-GPU paths of the solve: one process per GPU,
torch.distributed (NCCL over NVLink/NVSwitch) for the exchange.

Config 5 of BASELINE.json reuses one factorization for a 256-RHS block
solve (`solve_multi(fac, B)`, solve.py:37-42 of the reference).  The
substitution of different right-hand-side columns is independent, so the
block shards by COLUMN: every rank holds a factorization of the same
operator (factorize() is bitwise deterministic, so the replicas are
identical, tests/test_gpu_parity.py::test_factorize_bitwise_deterministic),
rank g substitutes columns [lo_g, hi_g) on its own GPU with the library's
multi-RHS kernels, and one all-gather assembles the n x q solution on every
rank.  No data-path exchange happens during the substitution itself.

The collective is the only host-visible step; the per-rank substitution is
`h2f_solve_dev` (include/h2f.h), so nothing here computes on the host.
"""
from __future__ import annotations

import numpy as np

__all__ = ["column_ranges", "solve_multi_sharded", "broadcast_arrays", "broadcast_factorization"]


def column_ranges(q, world):
    """Contiguous, balanced column blocks: the first q % world ranks get one
    extra column.  Returns [(lo, hi)] per rank, covering [0, q) in order."""
    if q < 0 or world < 1:
        raise ValueError("need q >= 0 and world >= 1")
    base, extra = divmod(q, world)
    out, lo = [], 0
    for g in range(world):
        hi = lo + base + (1 if g < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def _device_solver(fac):
    """Column-block substitution on this rank's GPU through the C ABI."""
    import ctypes as C

    import torch

    from . import _lib as L

    def run(b_block):  # torch float64 (n, w) on the library's device, C-order
        x = torch.empty_like(b_block)
        torch.cuda.current_stream(b_block.device).synchronize()  # b_block's copy -> library stream
        if b_block.numel():
            L.check(L.lib().h2f_solve_dev(fac.handle.ptr, C.c_void_p(b_block.data_ptr()),
                                          C.c_void_p(x.data_ptr()), int(b_block.shape[1])), "h2f_solve_dev")
        return x

    return run


def solve_multi_sharded(fac, B, group=None, solver=None, device=None):
    """solve_multi(fac, B) with B's columns sharded over the ranks of `group`.

    B: (n, q) host array (every rank passes the same B, or at least the same
    shape; only the local columns are read).  Returns the full (n, q)
    solution as a host array on every rank.  Same shape checks and
    ValueError message as solve_multi (solve.py:40-41).

    `solver` (tests only) replaces the per-rank GPU substitution with a
    callable on host tensors; the default is the library's device path.
    """
    import torch
    import torch.distributed as dist

    B = np.asarray(B, dtype=np.float64)
    if B.ndim != 2 or B.shape[0] != fac.n:
        raise ValueError(f"right-hand side must have shape ({fac.n}, q)")
    n, q = B.shape
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    ranges = column_ranges(q, world)
    lo, hi = ranges[rank]
    wmax = max(h - l for l, h in ranges)
    if solver is None:
        from . import _lib as L

        # the shard lives on the library's own device (LOCAL_RANK under torchrun)
        dev = device if device is not None else torch.device("cuda", L.device())
        run = _device_solver(fac)
    else:
        dev = torch.device("cpu")
        run = solver
    local = torch.from_numpy(np.ascontiguousarray(B[:, lo:hi])).to(dev)
    x_local = run(local) if hi > lo else local
    if world == 1:
        return x_local.cpu().numpy()
    # equal-size blocks for the collective: pad to the widest shard
    send = torch.zeros((n, wmax), dtype=torch.float64, device=dev)
    send[:, : hi - lo] = x_local
    parts = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(parts, send, group=group)
    out = np.empty((n, q), dtype=np.float64)
    for (l, h), p in zip(ranges, parts):
        out[:, l:h] = p[:, : h - l].cpu().numpy()
    return out


def broadcast_arrays(arrays, src=0, group=None, device=None):
    """Broadcast a dict of NumPy arrays (e.g. serialize.pack of a factor)
    from rank `src`; returns the dict on every rank.  One small object
    broadcast for the layout, then one tensor broadcast per array (over
    NCCL on `device`, or gloo on the CPU)."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    layout = [[(k, v.dtype.str, v.shape) for k, v in sorted(arrays.items())]] if rank == src else [None]
    dist.broadcast_object_list(layout, src=src, group=group)
    out = {}
    for key, dt, shape in layout[0]:
        nbytes = int(np.prod(shape, dtype=np.int64)) * np.dtype(dt).itemsize
        if rank == src:
            raw = np.ascontiguousarray(arrays[key]).reshape(-1).view(np.uint8)
            t = torch.from_numpy(raw.copy()).to(device) if device is not None else torch.from_numpy(raw.copy())
        else:
            t = torch.empty(nbytes, dtype=torch.uint8, device=device)
        if nbytes:
            dist.broadcast(t, src=src, group=group)
        out[key] = t.cpu().numpy().view(np.dtype(dt)).reshape(shape)
    return out


def broadcast_factorization(fac, src=0, group=None, device=None, tree=None):
    """Factor once on rank `src`, then give every rank the same factor (the
    replicated factor of the column-sharded multi-RHS solve):
    the source packs its device factor (serialize.pack), the others rebuild
    it from the broadcast arrays (serialize.unpack).  `fac` is ignored on the
    other ranks."""
    import torch.distributed as dist

    from .serialize import pack, unpack

    rank = dist.get_rank(group)
    arrays = pack(fac) if rank == src else {}
    got = broadcast_arrays(arrays, src=src, group=group, device=device)
    return fac if rank == src else unpack(got, tree if tree is not None else getattr(fac, "tree", None))
