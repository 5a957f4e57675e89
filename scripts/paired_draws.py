"""Paired backward-error draws: CPU oracle vs B200 path on IDENTICAL operators
(VERDICT r01 item 1a/1b), run on the GPU box (its host cores run the oracle).

    python scripts/paired_draws.py FAMILY N SEEDS OUT.jsonl [key=value ...] [jobs=J]

For every seed (0 = the unperturbed operator, s > 0 = the dense near field
multiplied by (1 + 1e-14 z), z ~ N(0,1) from default_rng(s), the recipe of
scripts/oracle_big.py / scripts/draws_probe.py):
  * the oracle (1 BLAS thread, one process per seed, J in parallel) factors and
    solves, recording its threshold decisions;
  * the device path factors with its own decisions ("own");
  * the device path factors with the oracle's decisions forced ("replay").
One JSON line per (seed, arm) with raw and refined backward errors.
"""
import json
import os
import subprocess
import sys
import time

import numpy as np

sys.path.insert(0, ".")

fam, n, seeds_arg, out = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
seeds = [int(s) for s in seeds_arg.split(",")]
over_args = [a for a in sys.argv[5:] if not a.startswith(("jobs=", "vmem_gb=", "replay="))]
do_replay = next((a.split("=")[1] for a in sys.argv[5:] if a.startswith("replay=")), "1") != "0"
jobs = int(next((a.split("=")[1] for a in sys.argv[5:] if a.startswith("jobs=")), "8"))
# per-oracle address-space cap (a runaway oracle dies alone instead of
# taking the box down)
vmem_gb = float(next((a.split("=")[1] for a in sys.argv[5:] if a.startswith("vmem_gb=")), "30"))
over = {}
for a in over_args:
    k, v = a.split("=")
    over[k] = float(v) if "." in v or "e" in v else int(v)
work = os.path.join("gpurun_out", f"paired_{fam}_{n}")
os.makedirs(work, exist_ok=True)
env = dict(os.environ, OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1", MKL_NUM_THREADS="1")

# ---- oracle processes (bounded parallelism) --------------------------------
pending = list(seeds)
running = {}
done = {}


def launch():
    while pending and len(running) < jobs:
        s = pending.pop(0)
        extra = [] if s == 0 else ["perturb=1e-14", f"seed={s}"]
        py = " ".join([sys.executable, "scripts/oracle_big.py", fam, str(n), f"{work}/orc_{s}.npz",
                       *over_args, *extra, f"decisions={work}/dec_{s}.npz"])
        cmd = ["bash", "-c", f"ulimit -v {int(vmem_gb * 1024 * 1024)}; exec nice -n 5 {py}"]
        log = open(f"{work}/orc_{s}.log", "w")
        running[s] = (subprocess.Popen(cmd, stdout=log, stderr=subprocess.STDOUT, env=env), log, time.time())


def poll():
    for s in list(running):
        p, log, t0 = running[s]
        if p.poll() is not None:
            log.close()
            done[s] = (p.returncode, time.time() - t0)
            del running[s]
    launch()


launch()

# ---- device arms -----------------------------------------------------------
import paper_2509_11152_b200 as H  # noqa: E402
from paper_2509_11152_b200 import _lib as L  # noqa: E402

tree, part, spec, h2, prm = H.build_problem(fam, n, **over)
base_dense = dict(h2.dense)
x_ref = np.random.Generator(np.random.Philox(7)).standard_normal(n)
fo = open(out, "a")


def operator(seed):
    if seed == 0:
        h2.dense = dict(base_dense)
    else:
        rng = np.random.default_rng(seed)
        dense = {}
        for key in sorted(base_dense):
            blk = base_dense[key]
            z = rng.standard_normal(blk.shape)
            if key[0] == key[1]:
                z = 0.5 * (z + z.T)
            dense[key] = blk * (1.0 + 1e-14 * z)
        h2.dense = dense
    object.__setattr__(h2, "_h2f_device", None)  # re-upload the operator
    return H.matvec(h2, x_ref)


def arm(seed, mode, b, dec=None):
    if dec is not None:
        L.replay_set(dec["kept"], dec["created"])
    try:
        t0 = time.perf_counter()
        fac = H.factorize(h2, prm["eps_lu"])
        tf = time.perf_counter() - t0
        stats = L.replay_stats() if dec is not None else None
    finally:
        if dec is not None:
            L.replay_clear()
    x0 = H.solve(fac, b)
    x = H.refined_solve(h2, fac, b, steps=1)
    nb = np.linalg.norm(b)
    row = {"arm": mode, "family": fam, "n": n, "seed": seed, "fact_s": round(tf, 2),
           "e_b_raw": float(np.linalg.norm(H.matvec(h2, x0) - b) / nb),
           "e_b": float(np.linalg.norm(H.matvec(h2, x) - b) / nb),
           "top": fac.top_size, "levels": [[r.level, r.nbatches, r.max_rank] for r in fac.records],
           "replay": stats}
    del fac
    fo.write(json.dumps(row) + "\n")
    fo.flush()
    print(json.dumps(row), flush=True)


for s in seeds:
    b = operator(s)
    arm(s, "own", b)
    poll()

replayed = set()
while len(replayed) < len(seeds):
    poll()
    ready = [s for s in done if s not in replayed]
    if not ready:
        time.sleep(5)
        continue
    for s in ready:
        replayed.add(s)
        rc, secs = done[s]
        summ = None
        try:
            with open(f"{work}/orc_{s}.log") as fh:
                summ = json.loads([ln for ln in fh if ln.startswith("{")][-1])
        except Exception:
            pass
        if rc != 0 or summ is None:
            fo.write(json.dumps({"arm": "oracle", "seed": s, "rc": rc, "failed": True}) + "\n")
            continue
        fo.write(json.dumps({"arm": "oracle", "family": fam, "n": n, "seed": s, "fact_s": summ["fact_s"],
                             "e_b_raw": summ["e_b_raw"], "e_b": summ["e_b"], "top": summ["top"],
                             "levels": summ["levels"], "wall_s": round(secs, 1)}) + "\n")
        fo.flush()
        if do_replay:
            b = operator(s)
            arm(s, "replay", b, np.load(f"{work}/dec_{s}.npz"))
fo.close()
