"""Device harness: the reference's measured pipeline
(/root/reference/pkg/src/h2factor/harness.py) with the factorization, the
solves and every matvec on the B200 path.

  ExperimentConfig.from_problem  harness.py:87-131 (same fields and rows)
  run(config)                    harness.py:197-249 -> report dict with the
                                 RunReport keys (+ "device", "profile")
  validate(config)               harness.py:252-308 (dense references, n <= oracle_cap)
  scaling_sweep / thread_sweep   harness.py:311-366
  write_outputs / write_sweep_outputs / write_thread_outputs
                                 harness.py:375-422 (same files, columns, formats)

The operator is built on the host exactly like the reference (problem.py);
timings are host wall clock around the public API calls, as in the
reference; the factorization's `phases` come from CUDA events on the
library stream.  With `profile=True` the report also carries per-kernel
device seconds, algorithmic flops/bytes and the achieved fraction of the
FP64 DMMA / HBM peaks (the roofline columns).  The dense references of
validate() are the checker (NumPy LAPACK on the host), as in the reference.

    python -m paper_2509_11152_b200.cli run --problem cov2d --n 16384
"""
from __future__ import annotations

import csv
import dataclasses
import hashlib
import json
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import __version__
from .factorization import factorize
from .h2core import matvec
from .problem import PROBLEMS, build_problem, entry_block, h2_nbytes, make_low_rank_factor
from .solve import refined_solve

__all__ = ["PROBLEMS", "ExperimentConfig", "run", "validate", "scaling_sweep", "thread_sweep",
           "write_outputs", "write_sweep_outputs", "write_thread_outputs"]

# phase keys of H2Factorization.phase_seconds -> report labels (harness.py:74-83)
PHASE_LABELS = {
    "norm": "norm_estimate",
    "extract": "block_extract",
    "color": "coloring",
    "augment": "basis_augmentation",
    "project": "projection",
    "partial_lu": "partial_lu",
    "transition": "level_transition",
    "top": "top_solve",
}


@dataclass
class ExperimentConfig:
    """One experiment (harness.py:87-131); `threads` is accepted for API
    parity (the device path batches clusters instead of using a pool)."""

    problem: str
    n: int
    m: int
    p0: int
    dim: int
    eta: float
    alpha_r: float
    eps: float
    eps_lu: float
    corr_length: float = 0.1
    kappa: float = 3.0
    lru_rank: int = 0
    refine_steps: int = 1
    threads: int = 1
    seed: int = 7
    deterministic: bool = True
    oracle_cap: int = 4096
    out: str | None = None
    # build the operator on the device (construct.py)
    # instead of the reference's host construction
    device_build: bool = False

    @classmethod
    def from_problem(cls, problem, n, **overrides):
        if problem not in PROBLEMS:
            raise ValueError(f"unknown problem {problem!r}; choose from {sorted(PROBLEMS)}")
        row = {k: v for k, v in PROBLEMS[problem].items() if k != "family"}
        row.setdefault("lru_rank", 0)
        row.update({k: v for k, v in overrides.items() if v is not None})
        return cls(problem=problem, n=n, **row)

    @property
    def family(self):
        return PROBLEMS[self.problem]["family"]

    def builder_overrides(self):
        keys = ("m", "p0", "dim", "eta", "alpha_r", "eps", "eps_lu", "corr_length", "kappa", "lru_rank", "seed")
        return {k: getattr(self, k) for k in keys}


def _operator(config):
    from . import problem as P
    if config.device_build:
        from .construct import build_problem_device
        tree, part, spec, h2, prm = build_problem_device(config.problem, config.n, **config.builder_overrides())
        bs = h2.build_seconds
        t = {"construction": bs["host_structure"] + bs["construction"], "compression": bs["compression"]}
        if "low_rank_update" in bs:
            t["low_rank_update"] = bs["low_rank_update"] + bs["compression_after_update"]
        return tree, spec, h2, prm, t
    tree, part, spec, h2, prm = build_problem(config.problem, config.n, **config.builder_overrides())
    return tree, spec, h2, prm, dict(P.LAST_BUILD_TIMINGS)


def _h2_bytes(h2):
    built = getattr(h2, "_h2f_built", None)
    return built.nbytes if built is not None else int(h2_nbytes(h2))


def _profile_columns(prof):
    """Roofline columns: per kernel family device seconds, algorithmic work
    and the achieved fraction of the bound (FP64 DMMA or HBM)."""
    from . import _lib as L
    try:
        with open(Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json") as fh:
            hbm = float(json.load(fh).get("hbm_gbs", 6550.0))
    except OSError:
        hbm = 6550.0
    dmma = L.bench_dmma(20000)
    ridge = dmma * 1e12 / (hbm * 1e9)
    cols = {}
    for name, p in sorted(prof.items(), key=lambda kv: -kv[1]["seconds"]):
        s = max(p["seconds"], 1e-12)
        ai = p["flops"] / max(p["bytes"], 1.0)
        tensor = ai >= ridge
        achieved = p["flops"] / s / 1e12 if tensor else p["bytes"] / s / 1e9
        cols[name] = {"seconds": p["seconds"], "launches": p["launches"], "gflop": p["flops"] / 1e9,
                      "gbytes": p["bytes"] / 1e9, "bound": "tensor" if tensor else "hbm",
                      "achieved": achieved, "unit": "TFLOP/s" if tensor else "GB/s",
                      "frac": achieved / (dmma if tensor else hbm)}
    return {"fp64_dmma_tflops": dmma, "hbm_gbs": hbm, "kernels": cols}


def run(config, profile=False, keep_solution=False):
    """Full pipeline for one configuration (harness.py:197-249)."""
    from . import _lib as L

    tree, spec, h2, prm, timings = _operator(config)
    if profile:
        L.profile_enable(True)
        L.profile_reset()
    t0 = time.perf_counter()
    fac = factorize(h2, config.eps_lu, threads=config.threads)
    timings["factorization"] = time.perf_counter() - t0
    x_ref = np.random.Generator(np.random.Philox(config.seed)).standard_normal(config.n)
    b = matvec(h2, x_ref)
    t0 = time.perf_counter()
    x = refined_solve(h2, fac, b, threads=config.threads, steps=config.refine_steps)
    timings["solve"] = time.perf_counter() - t0
    prof = L.profile_get() if profile else None
    if profile:
        L.profile_enable(False)
    e_b = float(np.linalg.norm(matvec(h2, x) - b) / np.linalg.norm(b))

    phases = {"construction": timings["construction"], "compression": timings["compression"]}
    if "low_rank_update" in timings:
        phases["low_rank_update"] = timings["low_rank_update"]
    for key, label in PHASE_LABELS.items():
        if key in fac.phase_seconds:
            phases[label] = fac.phase_seconds[key]
    phases["solve"] = timings["solve"]
    report = {
        "version": __version__,
        "device": "cuda",
        "config": dataclasses.asdict(config),
        "n": config.n,
        "e_b": e_b,
        "solution_digest": hashlib.sha256(x.tobytes()).hexdigest(),
        "h2_bytes": _h2_bytes(h2),
        "factor_bytes": int(fac.nbytes()),
        "kmax_construction": int(max(h2.rank.values())) if h2.rank else 0,
        "kmax_factorization": int(fac.max_rank()),
        "csp_max": int(max((r.csp for r in fac.records), default=0)),
        "timings": timings,
        "phases": phases,
        "levels": [{"level": r.level, "time_s": r.time_s, "csp": r.csp, "max_rank": r.max_rank}
                   for r in fac.records],
        "ranks": [r.max_rank for r in fac.records],
    }
    if profile:
        report["profile"] = _profile_columns(prof)
    if keep_solution:
        report["solution"] = x
    return report


def _dense_exact(tree, spec, n):
    idx = np.arange(n)
    return entry_block(spec, tree.points, idx, idx)


def validate(config):
    """Dense references at small n (harness.py:252-308): the compressed
    operator densified through the device matvec (identity block), and the
    exact kernel matrix (plus W W^T for the low-rank row), each solved by
    pivoted LU on the host; pass iff solution error <= 1e-4 and
    e_b <= 10 eps_lu against the densified operator."""
    if config.n > config.oracle_cap:
        raise ValueError(f"n={config.n} exceeds oracle cap {config.oracle_cap}")
    from scipy.linalg import lu_factor, lu_solve

    tree, spec, h2, prm, _ = _operator(config)
    fac = factorize(h2, config.eps_lu, threads=config.threads)
    x_ref = np.random.Generator(np.random.Philox(config.seed)).standard_normal(config.n)
    b = matvec(h2, x_ref)
    x = refined_solve(h2, fac, b, threads=config.threads, steps=config.refine_steps)
    e_b = float(np.linalg.norm(matvec(h2, x) - b) / np.linalg.norm(b))
    n = config.n
    dense_h2 = matvec(h2, np.eye(n))
    x_star = lu_solve(lu_factor(dense_h2), b)
    exact = _dense_exact(tree, spec, n)
    if config.lru_rank > 0:
        w = make_low_rank_factor(n, config.lru_rank, config.seed)
        exact = exact + w @ w.T
    x_exact = lu_solve(lu_factor(exact), b)
    sol = float(np.linalg.norm(x - x_star) / np.linalg.norm(x_star))
    result = {
        "e_b": e_b,
        "solution_error": sol,
        "solution_error_exact_kernel": float(np.linalg.norm(x - x_exact) / np.linalg.norm(x_exact)),
        "compression_error": float(np.linalg.norm(dense_h2 - exact) / np.linalg.norm(exact)),
        "tol_solution": 1e-4,
        "tol_backward": 10.0 * config.eps_lu,
    }
    result["passed"] = bool(sol <= result["tol_solution"] and e_b <= result["tol_backward"])
    return result


def _slope(xs, ys):
    return float(np.polyfit(np.log(xs), np.log(ys), 1)[0])


def scaling_sweep(problem, sizes, **overrides):
    """Runs over sizes with fitted log-log slopes (harness.py:311-343)."""
    if len(sizes) < 3:
        raise ValueError("scaling sweep needs at least three sizes")
    rows = []
    for n in sizes:
        rep = run(ExperimentConfig.from_problem(problem, n, **overrides))
        rows.append({"n": n, "construction_s": rep["timings"]["construction"],
                     "compression_s": rep["timings"]["compression"],
                     "factorization_s": rep["timings"]["factorization"], "solve_s": rep["timings"]["solve"],
                     "h2_bytes": rep["h2_bytes"], "factor_bytes": rep["factor_bytes"], "e_b": rep["e_b"]})
    ns = [r["n"] for r in rows]
    slopes = {"factorization_time": _slope(ns, [r["factorization_s"] for r in rows]),
              "solve_time": _slope(ns, [r["solve_s"] for r in rows]),
              "factor_memory": _slope(ns, [r["factor_bytes"] for r in rows])}
    return {"rows": rows, "slopes": slopes}


def thread_sweep(problem, n, thread_list, **overrides):
    """One configuration across `threads` values (harness.py:346-366); the
    device result is the same bits for every value."""
    if any(t < 1 for t in thread_list):
        raise ValueError("thread counts must be positive")
    rows = []
    for threads in thread_list:
        rep = run(ExperimentConfig.from_problem(problem, n, threads=threads, **overrides))
        rows.append({"threads": threads, "factorization_s": rep["timings"]["factorization"],
                     "solve_s": rep["timings"]["solve"], "e_b": rep["e_b"],
                     "solution_digest": rep["solution_digest"], "factor_bytes": rep["factor_bytes"]})
    for row in rows:
        row["speedup"] = rows[0]["factorization_s"] / row["factorization_s"]
    return rows


def _fmt(v):
    return f"{v:.6e}" if isinstance(v, float) else str(v)


def _report_json(report):
    return {k: v for k, v in report.items() if k != "solution"}


def write_outputs(report, out_dir):
    """report.json, levels.csv, phases.csv (harness.py:375-394)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    with open(out / "report.json", "w", encoding="utf-8") as fh:
        json.dump(_report_json(report), fh, indent=2)
        fh.write("\n")
    with open(out / "levels.csv", "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(["level", "time_s", "csp", "max_rank"])
        for r in report["levels"]:
            w.writerow([r["level"], _fmt(float(r["time_s"])), r["csp"], r["max_rank"]])
    total = sum(report["phases"].values())
    with open(out / "phases.csv", "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(["phase", "time_s", "fraction"])
        for name, sec in report["phases"].items():
            w.writerow([name, _fmt(float(sec)), _fmt(float(sec / total if total > 0 else 0.0))])
    if "profile" in report:
        with open(out / "roofline.csv", "w", newline="", encoding="utf-8") as fh:
            w = csv.writer(fh)
            w.writerow(["kernel", "seconds", "launches", "gflop", "gbytes", "bound", "achieved", "unit", "frac"])
            for name, c in report["profile"]["kernels"].items():
                w.writerow([name, _fmt(float(c["seconds"])), c["launches"], _fmt(float(c["gflop"])),
                            _fmt(float(c["gbytes"])), c["bound"], _fmt(float(c["achieved"])), c["unit"],
                            _fmt(float(c["frac"]))])


def write_sweep_outputs(sweep, out_dir):
    """sweep.csv, slopes.json (harness.py:397-410)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    rows = sweep["rows"]
    with open(out / "sweep.csv", "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(list(rows[0]))
        for r in rows:
            w.writerow([_fmt(r[k]) for k in rows[0]])
    with open(out / "slopes.json", "w", encoding="utf-8") as fh:
        json.dump(sweep["slopes"], fh, indent=2)
        fh.write("\n")


def write_thread_outputs(rows, out_dir):
    """threads.csv (harness.py:413-422)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    with open(out / "threads.csv", "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(list(rows[0]))
        for r in rows:
            w.writerow([_fmt(r[k]) for k in rows[0]])
