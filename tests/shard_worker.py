"""One rank of the subtree-sharded factorization check (tests/test_gpu_sharded.py).

Launched by torch.distributed.run with the gloo backend; every rank runs
factorize_sharded on the same operator, exports a digest of its (replicated)
factor, and rank 0 compares every rank's digest with the single-GPU
factorize() of the same operator: batches, kept/redundant counts, fill events
and a SHA-256 over every Q~, LU, pivot, eliminator block and the top LU must
be identical, and so must the refined solution.  Several ranks may share one
GPU here: each has its own library context and the ranks only meet in host
collectives (no kernel waits on another process).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
        --master-port 29600 tests/shard_worker.py cov2d 4096 out.json
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2509_11152_b200 as H  # noqa: E402
from paper_2509_11152_b200 import multigpu as MG  # noqa: E402
from paper_2509_11152_b200 import problem as P  # noqa: E402


def digest(fac):
    h = hashlib.sha256()
    recs = []
    for rec in fac.records:
        rs = {"level": rec.level, "batches": rec.batches, "up": rec.up_index.tolist(),
              "fills": rec.fill_events(), "r": [], "edges": []}
        for c in rec.clusters:
            f = rec.factors[c]
            rs["r"].append(int(f.r))
            h.update(np.ascontiguousarray(f.q).tobytes())
            if f.r:
                h.update(np.ascontiguousarray(f.lu).tobytes())
                h.update(f.piv.tobytes())
            for o, k, m in f.edges:
                rs["edges"].append([int(o), k, list(m.shape)])
                h.update(np.ascontiguousarray(m).tobytes())
            f._q = f._lu = f._piv = f._edges = None  # keep host memory flat
        recs.append(rs)
    h.update(np.ascontiguousarray(fac.top_lu).tobytes())
    h.update(np.ascontiguousarray(fac.top_piv).tobytes())
    return {"records": recs, "sha": h.hexdigest(), "nbytes": int(fac.nbytes()), "top_size": fac.top_size,
            "eps_fill": fac.eps_fill}


def main():
    name, n, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    over = json.loads(sys.argv[4]) if len(sys.argv) > 4 else {}
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    tree, part, spec, h2, prm = P.build_problem(name, n, **over)
    xr = P.rhs_for(h2)
    b = H.matvec(h2, xr)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    fac = MG.factorize_sharded(h2, prm["eps_lu"])
    t_shard = time.perf_counter() - t0
    stats = MG.shard_stats()
    stats["wall_s"] = t_shard
    x = H.refined_solve(h2, fac, b, steps=1)
    d = digest(fac)
    d["x_sha"] = hashlib.sha256(x.tobytes()).hexdigest()
    d["stats"] = stats
    del fac  # the single-GPU reference factor below needs the memory
    got = [None] * world
    dist.all_gather_object(got, d)
    if rank == 0:
        t0 = time.perf_counter()
        ref = H.factorize(h2, prm["eps_lu"])
        t_single = time.perf_counter() - t0
        dr = digest(ref)
        xs = H.refined_solve(h2, ref, b, steps=1)
        dr["x_sha"] = hashlib.sha256(xs.tobytes()).hexdigest()
        res = {"case": [name, n, over], "world": world, "ranks": [], "single_wall_s": t_single}
        for g, dg in enumerate(got):
            res["ranks"].append({
                "rank": g,
                "structure_equal": dg["records"] == dr["records"],
                "values_equal": dg["sha"] == dr["sha"],
                "solution_equal": dg["x_sha"] == dr["x_sha"],
                "nbytes_equal": dg["nbytes"] == dr["nbytes"] and dg["top_size"] == dr["top_size"],
                "stats": dg["stats"],
            })
        res["e_b"] = float(np.linalg.norm(H.matvec(h2, x) - b) / np.linalg.norm(b))
        with open(out, "w") as fh:
            json.dump(res, fh, indent=1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
