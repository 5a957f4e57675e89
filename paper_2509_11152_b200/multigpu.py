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

The factorization itself shards by cluster-tree SUBTREE
(`factorize_sharded`, h2f_factorize_sharded): rank g owns the clusters below
its run of top-level clusters; the per-batch exchange (Q~ and eliminator
panels to the holders of neighbour blocks, max-reduced kept counts / pivot
status / fill norms) runs through the h2f_comm callbacks that `TorchComm`
binds to torch.distributed -- NCCL on device buffers over NVLink, or gloo
staged through host memory (tests).  The result is the single-GPU factor,
bit for bit, replicated on every rank.
"""
from __future__ import annotations

import numpy as np

__all__ = ["column_ranges", "solve_multi_sharded", "broadcast_arrays", "broadcast_factorization",
           "TorchComm", "factorize_sharded", "shard_owners", "shard_stats"]


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


# --------------------------------------------------------------------------
# subtree-sharded factorization (factorization.py:433-505)
# --------------------------------------------------------------------------

class _DevBytes:
    """A raw device range as a CUDA-array-interface object (zero-copy view
    for torch.as_tensor)."""

    def __init__(self, addr, nbytes, typestr="|u1", itemsize=1):
        self.__cuda_array_interface__ = {"shape": (nbytes // itemsize,), "typestr": typestr,
                                         "data": (int(addr), False), "version": 3, "strides": None}


class TorchComm:
    """The h2f_comm callbacks (include/h2f.h) over a torch.distributed group.

    NCCL: the library's device buffers are wrapped zero-copy and the
    collectives run on torch's current stream, synchronised before
    returning (the library drained its own stream before the call).  gloo:
    the same collectives staged through host memory (CPU tests, or a box
    without NCCL).  A Python exception inside a callback becomes a nonzero
    return code, and `reraise()` raises it after the library call."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        from . import _lib as L

        self._torch, self._dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"
        self.device = torch.device("cuda", L.device()) if self.nccl else None
        self.error = None
        self.seconds = 0.0
        self._fns = (L.ALLREDUCE_FN(self._wrap(self._allreduce_max)),
                     L.ALLREDUCE_DEV_FN(self._wrap(self._allreduce_sum_dev)),
                     L.ALLTOALLV_FN(self._wrap(self._alltoallv_dev)),
                     L.BROADCAST_FN(self._wrap(self._broadcast_dev)))
        self.struct = L.Comm(self.rank, self.world, None, *self._fns)

    def _wrap(self, fn):
        def cb(*args):
            try:
                fn(*args[1:])
                return 0
            except BaseException as e:  # noqa: BLE001 -- must not unwind through C
                if self.error is None:
                    self.error = e
                return 1
        return cb

    def reraise(self):
        if self.error is not None:
            e, self.error = self.error, None
            raise e

    def _dev_view(self, addr, nbytes, dtype):
        torch = self._torch
        item = 8 if dtype == torch.float64 else 1
        obj = _DevBytes(addr, nbytes, "<f8" if item == 8 else "|u1", item)
        return torch.as_tensor(obj, device=torch.device("cuda", torch.cuda.current_device())
                               if self.device is None else self.device)

    def _sync(self):
        if self.nccl:
            self._torch.cuda.current_stream(self.device).synchronize()

    def _src(self, root):
        return root if self.group is None else self._dist.get_global_rank(self.group, root)

    def _allreduce_max(self, buf, n):
        torch, dist = self._torch, self._dist
        host = torch.from_numpy(np.ctypeslib.as_array(buf, (n,)))
        if self.nccl:
            t = host.to(self.device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
            host.copy_(t.cpu())
        else:
            dist.all_reduce(host, op=dist.ReduceOp.MAX, group=self.group)

    def _allreduce_sum_dev(self, addr, n):
        torch, dist = self._torch, self._dist
        t = self._dev_view(addr, 8 * n, torch.float64)
        if self.nccl:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
            self._sync()
        else:
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
            t.copy_(h)
            torch.cuda.synchronize(t.device)

    def _alltoallv_dev(self, send, send_counts, recv, recv_counts):
        torch, dist = self._torch, self._dist
        sc = [int(send_counts[g]) for g in range(self.world)]
        rc = [int(recv_counts[g]) for g in range(self.world)]
        st = self._dev_view(send, max(sum(sc), 1), torch.uint8)[: sum(sc)]
        rt = self._dev_view(recv, max(sum(rc), 1), torch.uint8)[: sum(rc)]
        if self.nccl:
            dist.all_to_all_single(rt, st, rc, sc, group=self.group)
            self._sync()
        else:
            hr = torch.empty(sum(rc), dtype=torch.uint8)
            dist.all_to_all_single(hr, st.cpu(), rc, sc, group=self.group)
            rt.copy_(hr)
            torch.cuda.synchronize(rt.device)

    def _broadcast_dev(self, addr, nbytes, root):
        torch, dist = self._torch, self._dist
        t = self._dev_view(addr, nbytes, torch.uint8)
        if self.nccl:
            dist.broadcast(t, src=self._src(root), group=self.group)
            self._sync()
        else:
            h = t.cpu() if self.rank == root else torch.empty(nbytes, dtype=torch.uint8)
            dist.broadcast(h, src=self._src(root), group=self.group)
            if self.rank != root:
                t.copy_(h)
                torch.cuda.synchronize(t.device)


def factorize_sharded(h2, eps_lu, threads=1, norm_estimate=None, group=None):
    """factorize(h2, eps_lu) split over the ranks of `group` by cluster-tree
    subtree (h2f_factorize_sharded).  Every rank passes the same operator;
    every rank returns the complete factor, identical to the single-GPU
    factorize() (batches, kept counts, fill, pivots and values)."""
    del threads
    from .factorization import factorize_with

    return factorize_with(h2, eps_lu, norm_estimate, comm=TorchComm(group))


def shard_owners(tree, top_level, world):
    """Owner rank per cluster-tree node for a world-way subtree split
    (h2f_shard_owners; host-only).  -1 above the top level."""
    from . import _lib as L

    parent = np.ascontiguousarray(tree.parent, dtype=np.int64)
    level = np.ascontiguousarray(tree.level, dtype=np.int64)
    out = np.empty(len(parent), dtype=np.int32)
    L.check(L.lib().h2f_shard_owners(len(parent), L.ptr(parent, L.i64p), L.ptr(level, L.i64p),
                                     -1 if top_level is None else int(top_level), int(world),
                                     L.ptr(out, L.i32p)), "h2f_shard_owners")
    return out


def shard_stats():
    """Counters of this process's last sharded factorization (dict)."""
    from . import _lib as L

    v = np.zeros(8)
    L.check(L.lib().h2f_shard_stats(L.ptr(v)), "h2f_shard_stats")
    keys = ("clusters_here", "clusters_total", "bytes_sent", "collectives", "schur_tiles_here", "batches",
            "collective_seconds", "gather_bytes")
    return dict(zip(keys, v.tolist()))
