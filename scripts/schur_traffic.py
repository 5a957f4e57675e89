"""One config-2 factorization with the per-launch profiler log on (H2F_PROF_LOG),
meant to run under ncu filtered to the Schur-complement GEMM symbols
(role 1): pairs every Schur launch's ncu DRAM bytes with the library's
algorithmic bytes and flops for the same launch (bench.py roofline.traffic).

    H2F_PROF_LOG=gpurun_out/prof.log ncu --kernel-name regex:gemm_schur \\
        --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \\
        --log-file gpurun_out/schur_ncu.csv python scripts/schur_traffic.py
    python scripts/schur_traffic.py --summarize gpurun_out/prof.log gpurun_out/schur_ncu.csv OUT.json
"""
import csv
import json
import sys

import numpy as np

sys.path.insert(0, ".")


def run():
    import bench
    import paper_2509_11152_b200 as H
    from paper_2509_11152_b200 import _lib as L
    cfg = bench.CONFIGS[2]
    tree, part, spec, h2, prm = H.build_problem(cfg["problem"], cfg["n"], **cfg["over"])
    L.ensure_init()
    L.profile_enable(True)
    fac = H.factorize(h2, prm["eps_lu"])
    L.profile_get()
    print("factorized", fac.top_size)


def summarize(prof_log, ncu_csv, out):
    alg = []
    for line in open(prof_log):
        p = line.split()
        if p and p[0] == "gemm_schur":
            alg.append((float(p[1]), float(p[2]), float(p[4])))  # flops, bytes, ms (events)
    rows = [r for r in csv.reader(open(ncu_csv)) if len(r) > 10]
    hdr = rows[0]
    ik, iid = hdr.index("Kernel Name"), hdr.index("ID")
    im, iv = hdr.index("Metric Name"), hdr.index("Metric Value")
    per = {}
    for r in rows[1:]:
        d = per.setdefault(int(r[iid]), {"kernel": r[ik]})
        d[r[im]] = float(r[iv].replace(",", ""))
    launches = [per[k] for k in sorted(per)]
    n = min(len(alg), len(launches))
    dram = np.array([l["dram__bytes_read.sum"] + l["dram__bytes_write.sum"] for l in launches[:n]])
    dur = np.array([l["gpu__time_duration.sum"] for l in launches[:n]])  # ns
    fl = np.array([a[0] for a in alg[:n]])
    by = np.array([a[1] for a in alg[:n]])
    res = {"launches_ncu": len(launches), "launches_profiler": len(alg), "paired": n,
           "dram_bytes_per_launch": float(dram.mean()), "algorithmic_bytes_per_launch": float(by.mean()),
           "traffic_over_algorithmic": float(dram.sum() / by.sum()),
           "flops_per_launch": float(fl.mean()),
           "ncu_serialised_tflops": float(fl.sum() / (dur.sum() * 1e-9) / 1e12),
           "ncu_time_s": float(dur.sum() * 1e-9),
           "by_kernel": {}}
    for name in sorted(set(l["kernel"] for l in launches[:n])):
        idx = [i for i in range(n) if launches[i]["kernel"] == name]
        res["by_kernel"][name] = {"launches": len(idx), "dram_over_alg": float(dram[idx].sum() / by[idx].sum()),
                                  "time_s": float(dur[idx].sum() * 1e-9)}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--summarize":
        summarize(*sys.argv[2:5])
    else:
        run()
