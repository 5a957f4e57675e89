"""World-size-2 gloo tests of the column-sharded multi-RHS solve
(paper_2509_11152_b200/multigpu.py, BASELINE config 5).

The per-rank substitution is injected (the CPU oracle's substitute) so the
host logic -- column ranges, padding of ragged shards, the all-gather and
the reassembly -- runs here without a GPU.  The GPU path of the same
function is covered by tests/test_gpu_parity.py::test_solve_multi_sharded_single_rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2509_11152_b200.multigpu import column_ranges


def test_column_ranges_cover_and_balance():
    for q in [0, 1, 7, 8, 255, 256, 257]:
        for world in [1, 2, 3, 8]:
            rg = column_ranges(q, world)
            assert len(rg) == world
            assert rg[0][0] == 0 and rg[-1][1] == q
            assert all(a[1] == b[0] for a, b in zip(rg, rg[1:]))
            widths = [h - l for l, h in rg]
            assert max(widths) - min(widths) <= 1
    assert column_ranges(256, 8)[3] == (96, 128)
    with pytest.raises(ValueError):
        column_ranges(4, 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from threadpoolctl import threadpool_limits

    from golden_util import problem
    from oracle import h2_oracle as O
    from paper_2509_11152_b200.multigpu import solve_multi_sharded

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _, _, _, h2, prm = problem("cov2d_1024")
        with threadpool_limits(1):
            fac = O.factorize(h2, prm["eps_lu"])
        B = np.random.default_rng(11).standard_normal((h2.n, q))
        seen = []

        def solver(block):
            seen.append(block.shape[1])
            with threadpool_limits(1):
                return torch.from_numpy(O.substitute(fac, block.numpy()))

        X = solve_multi_sharded(fac, B, solver=solver)
        np.save(os.path.join(out_dir, f"x{rank}.npy"), X)
        np.save(os.path.join(out_dir, f"w{rank}.npy"), np.array(seen))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("q", [5, 8])
def test_solve_multi_sharded_gloo_world2(tmp_path, q):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), q, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    from threadpoolctl import threadpool_limits

    from golden_util import problem
    from oracle import h2_oracle as O

    _, _, _, h2, prm = problem("cov2d_1024")
    with threadpool_limits(1):
        fac = O.factorize(h2, prm["eps_lu"])
        B = np.random.default_rng(11).standard_normal((h2.n, q))
        # per-shard substitution (BLAS blocking depends on the block width)
        X_ref = np.hstack([O.substitute(fac, B[:, l:h]) for l, h in column_ranges(q, world)])
        X_full = O.substitute(fac, B)
    widths = [int(np.load(tmp_path / f"w{r}.npy")[0]) for r in range(world)]
    assert widths == [h - l for l, h in column_ranges(q, world)]
    for r in range(world):
        X = np.load(tmp_path / f"x{r}.npy")
        # every rank holds the assembled solution, bit-identical to the shards
        assert np.array_equal(X, X_ref)
        assert np.allclose(X, X_full, rtol=0, atol=1e-12 * np.abs(X_full).max())


def _bcast_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2509_11152_b200.multigpu import broadcast_arrays

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(4)
        src = {"meta": np.array('{"format": "x"}'), "q": rng.standard_normal((7, 5)),
               "piv": np.arange(9, dtype=np.int32), "empty": np.zeros(0), "ids": np.arange(4, dtype=np.int64)}
        got = broadcast_arrays(src if rank == 1 else {}, src=1)
        np.savez(os.path.join(out_dir, f"bc{rank}.npz"), **got)
    finally:
        dist.destroy_process_group()


def test_broadcast_arrays_gloo_world2(tmp_path):
    """The wire half of broadcast_factorization (serialize.pack arrays from
    one rank to all): dtypes, shapes, empty arrays and strings survive."""
    port = _free_port()
    mp.spawn(_bcast_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    q = np.random.default_rng(4).standard_normal((7, 5))
    for rank in range(2):
        with np.load(tmp_path / f"bc{rank}.npz") as z:
            assert np.array_equal(z["q"], q)
            assert str(z["meta"]) == '{"format": "x"}'
            assert z["piv"].dtype == np.int32 and np.array_equal(z["piv"], np.arange(9))
            assert z["empty"].shape == (0,) and np.array_equal(z["ids"], np.arange(4))


# ---------------------------------------------------------------- subtree sharding
# (h2f_factorize_sharded): the host-side pieces -- the owner
# map and the host collectives of TorchComm -- on CPU with gloo.  The device
# collectives and the sharded factorization itself: tests/test_gpu_sharded.py.

def test_shard_owners_are_contiguous_subtrees():
    import paper_2509_11152_b200 as H
    from paper_2509_11152_b200.multigpu import shard_owners

    for name, n, over in [("cov2d", 4096, {}), ("helmholtz3d", 16384, {"kappa": 0.0})]:
        pts, _ = H.generate_uniform_grid(n, 2 if name == "cov2d" else 3)
        tree = H.build_cluster_tree(pts, 64)
        part = H.dual_tree_traversal(tree, 0.9 if name == "cov2d" else 0.7)
        top = part.top_level
        for world in [1, 2, 4, 8]:
            own = shard_owners(tree, top, world)
            lv = np.asarray(tree.level)
            assert (own[lv < top] == -1).all() if world > 1 else (own == 0).all()
            if world == 1:
                continue
            tops = np.flatnonzero(lv == top)
            # contiguous, balanced runs of the top-level clusters
            assert list(own[tops]) == sorted(own[tops])
            assert np.bincount(own[tops], minlength=world).min() == len(tops) // world
            # every deeper cluster follows its parent
            deep = np.flatnonzero(lv > top)
            assert (own[deep] == own[np.asarray(tree.parent)[deep]]).all()
            # the leaves split evenly
            leaves = np.flatnonzero(lv == tree.depth)
            cnt = np.bincount(own[leaves], minlength=world)
            assert cnt.max() - cnt.min() <= 1 + len(leaves) // len(tops)


def test_shard_owners_rejects_too_many_ranks():
    import paper_2509_11152_b200 as H
    from paper_2509_11152_b200.multigpu import shard_owners

    pts, _ = H.generate_uniform_grid(4096, 2)
    tree = H.build_cluster_tree(pts, 64)
    part = H.dual_tree_traversal(tree, 0.9)
    ntop = int(np.count_nonzero(np.asarray(tree.level) == part.top_level))
    with pytest.raises(ValueError, match="top level"):
        shard_owners(tree, part.top_level, ntop + 1)
    with pytest.raises(ValueError, match="compressed level"):
        shard_owners(tree, None, 2)


def _comm_worker(rank, world, port, out_dir):
    import ctypes as C

    import torch.distributed as dist

    from paper_2509_11152_b200 import _lib as L
    from paper_2509_11152_b200.multigpu import TorchComm

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm()
        assert (comm.rank, comm.world, comm.nccl) == (rank, world, False)
        # the kept / pivot-status / fill-norm reduction: element-wise max,
        # -1 where a rank did not compute the candidate
        v = np.array([-1.0, 3.0 * rank, 0.5, -1.0 if rank else 7.25])
        rc = comm.struct.allreduce_max(None, v.ctypes.data_as(L.f64p), len(v))
        assert rc == 0
        np.save(os.path.join(out_dir, f"max{rank}.npy"), v)
        # a failing collective returns nonzero and re-raises after the call
        rc = comm.struct.allreduce_max(None, C.cast(None, L.f64p), 3)
        assert rc != 0
        with pytest.raises(Exception):
            comm.reraise()
    finally:
        dist.destroy_process_group()


def test_torchcomm_host_reduction_gloo(tmp_path):
    port = _free_port()
    mp.spawn(_comm_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"max{r}.npy"), [-1.0, 3.0, 0.5, 7.25])
