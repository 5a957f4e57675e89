"""Subtree-sharded factorization (h2f_factorize_sharded)
against the single-GPU factorize(): identical batches, kept/redundant counts,
fill events, values (SHA-256 over every Q~, LU, pivot, eliminator block and
the top LU) and refined solution, on every rank.  The ranks (2 or 4 gloo
processes, tests/shard_worker.py) share the test box's one GPU: each has its
own library context, exchanges go device -> host -> gloo -> device, and no
kernel ever waits on another process."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = [
    ("cov2d", 4096, {}, 2),
    ("cov2d", 4096, {}, 4),
    ("helmholtz3d", 4096, {"kappa": 0.0}, 2),
    ("helmholtz3d", 16384, {"kappa": 0.0}, 4),
    ("cov3d", 4096, {"eps_lu": 1e-8}, 2),
    ("helmholtz3d", 4096, {"dim": 2, "p0": 8, "eta": 0.9}, 2),
]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,n,over,world", CASES, ids=[f"{c[0]}_{c[1]}_{c[3]}r" for c in CASES])
def test_sharded_factor_is_the_single_gpu_factor(tmp_path, name, n, over, world):
    out = tmp_path / "res.json"
    env = dict(os.environ, H2F_DEVICE="0", H2F_ARENA_GB="6", OMP_NUM_THREADS="4")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(HERE, "shard_worker.py"), name, str(n), str(out), json.dumps(over)]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    r = json.loads(out.read_text())
    assert len(r["ranks"]) == world
    here = 0
    for rk in r["ranks"]:
        assert rk["structure_equal"], rk
        assert rk["values_equal"], rk
        assert rk["solution_equal"], rk
        assert rk["nbytes_equal"], rk
        st = rk["stats"]
        assert 0 < st["clusters_here"] < st["clusters_total"]
        here += st["clusters_here"]
    # every cluster is eliminated by exactly one rank
    assert here == r["ranks"][0]["stats"]["clusters_total"]


def test_torchcomm_device_collectives_nccl_single_rank():
    """The NCCL side of TorchComm (what bench.py --gpus N uses over NVLink):
    zero-copy views of library-style device buffers through every callback,
    at world size 1 on this one-GPU box; plus the degenerate sharded
    factorization (world 1) equal to factorize()."""
    import ctypes as C

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2509_11152_b200 as H
    from paper_2509_11152_b200 import _lib as L
    from paper_2509_11152_b200 import problem as P
    from paper_2509_11152_b200.multigpu import TorchComm, factorize_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        comm = TorchComm()
        assert comm.nccl and comm.world == 1
        a = torch.arange(10, dtype=torch.float64, device="cuda")
        assert comm.struct.allreduce_sum_dev(None, C.c_void_p(a.data_ptr()), 10) == 0
        assert torch.equal(a.cpu(), torch.arange(10, dtype=torch.float64))
        send = torch.arange(40, dtype=torch.uint8, device="cuda")
        recv = torch.zeros(40, dtype=torch.uint8, device="cuda")
        cnt = (C.c_int64 * 1)(40)
        assert comm.struct.alltoallv_dev(None, C.c_void_p(send.data_ptr()), cnt, C.c_void_p(recv.data_ptr()),
                                         cnt) == 0
        assert torch.equal(recv, send)
        assert comm.struct.broadcast_dev(None, C.c_void_p(recv.data_ptr()), 40, 0) == 0
        assert torch.equal(recv, send)
        v = np.array([1.0, -2.0])
        assert comm.struct.allreduce_max(None, v.ctypes.data_as(L.f64p), 2) == 0
        assert list(v) == [1.0, -2.0]
        comm.reraise()
        _, _, _, h2, prm = P.build_problem("cov2d", 4096)
        f1 = factorize_sharded(h2, prm["eps_lu"])
        f0 = H.factorize(h2, prm["eps_lu"])
        assert [r.batches for r in f1.records] == [r.batches for r in f0.records]
        assert np.array_equal(f1.top_lu, f0.top_lu)
    finally:
        dist.destroy_process_group()
