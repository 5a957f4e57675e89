"""Time factorize + refined_solve on the GPU across sizes (dev probe)."""
import sys, time, json
import numpy as np
sys.path.insert(0, '.')
import paper_2509_11152_b200 as H
from paper_2509_11152_b200 import _lib

cases = [a.split(':') for a in sys.argv[1:]] or [["cov2d", "16384"]]
for item in cases:
    name, n = item[0], int(item[1])
    over = {}
    for kv in item[2:]:
        k, v = kv.split('=')
        over[k] = float(v) if '.' in v or 'e' in v else int(v)
    t0 = time.perf_counter()
    tree, part, spec, h2, prm = H.build_problem(name, n, **over)
    tb = time.perf_counter() - t0
    t0 = time.perf_counter()
    fac = H.factorize(h2, prm["eps_lu"])
    tf = time.perf_counter() - t0
    _lib.profile_enable(True); _lib.profile_reset()
    t0 = time.perf_counter()
    fac2 = H.factorize(h2, prm["eps_lu"])
    tf2 = time.perf_counter() - t0
    prof = _lib.profile_get(); _lib.profile_enable(False)
    x_ref = np.random.Generator(np.random.Philox(7)).standard_normal(n)
    b = H.matvec(h2, x_ref)
    t0 = time.perf_counter()
    x = H.refined_solve(h2, fac2, b)
    ts = time.perf_counter() - t0
    _lib.profile_enable(True); _lib.profile_reset()
    t0 = time.perf_counter()
    x = H.refined_solve(h2, fac2, b)
    ts2 = time.perf_counter() - t0
    sprof = _lib.profile_get(); _lib.profile_enable(False)
    eb = np.linalg.norm(H.matvec(h2, x) - b) / np.linalg.norm(b)
    x0 = H.solve(fac2, b)
    eb0 = np.linalg.norm(H.matvec(h2, x0) - b) / np.linalg.norm(b)
    print(json.dumps({"case": f"{name}_{n}", "over": over, "build_s": round(tb, 2), "fact_s_first": round(tf, 4),
        "fact_s": round(tf2, 4), "solve_s_first": round(ts, 4), "solve_s": round(ts2, 4), "e_b": eb, "e_b_raw": eb0,
        "top": fac2.top_size, "nbytes_MB": fac2.nbytes() / 1e6,
        "batches": sum(r.nbatches for r in fac2.records),
        "phases": {k: round(v, 4) for k, v in fac2.phase_seconds.items()},
        "levels": [(r.level, round(r.time_s, 4), r.nbatches, r.max_rank) for r in fac2.records],
        "mem": _lib.memory_stats(),
        "kernels": {k: [round(v["seconds"], 4), v["launches"], round(v["flops"] / max(v["seconds"], 1e-12) / 1e9, 1)]
                    for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["seconds"])},
        "solve_kernels": {k: [round(v["seconds"], 4), v["launches"], round(v["bytes"] / max(v["seconds"], 1e-12) / 1e9, 1)]
                    for k, v in sorted(sprof.items(), key=lambda kv: -kv[1]["seconds"])}}), flush=True)
