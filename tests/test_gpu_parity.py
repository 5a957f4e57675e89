"""GPU parity: the B200 path (through the C ABI) against the CPU oracle and
the reference's golden fixtures.

Contract:
  * bit-exact integer structure (batches, r per cluster, offsets, up_index,
    edge (other, kind, shape), colouring statistics, top size, nbytes) for
    the families whose threshold decisions are robust (cov2d, cov3d);
  * norm estimate within 1e-12 relative (power iteration, reordered sums);
  * refined solution within 1e-8 relative of the reference's, backward error
    within 10x of the reference's (raw and refined);
  * skeleton projectors q[:, r:] q[:, r:]^T within 1e-10 of the oracle's.
"""
import numpy as np
import pytest

import paper_2509_11152_b200 as H
from golden_util import golden_structure, load, one_thread, problem, rhs, structure_of
from oracle import h2_oracle as O

pytestmark = pytest.mark.gpu

ROBUST = ["cov2d_1024", "cov3d_2048", "cov2d_4096", "cov3d_e8_4096", "cov2d_16384", "cov3d_e8_16384"]
SENSITIVE = ["laplace2d_2048", "helmholtz3d_2048", "laplace3d_4096", "osc2d_4096", "laplace3d_16384",
             "lru_cov3d_4096", "osc2d_65536"]
# cases whose backward error is chaotic for the reference itself: rounding-
# level (1e-14) perturbations of the operator move the reference's own e_b by
# decades (tests/golden/*_draws.json), so one draw is compared as a
# distribution (test_backward_error_distribution_chaotic), not pointwise
CHAOTIC = ["osc2d_65536"]

_fac_cache = {}


def gpu_factor(case):
    if case not in _fac_cache:
        _, _, _, h2, prm = problem(case)
        _fac_cache[case] = (h2, prm, H.factorize(h2, prm["eps_lu"]))
    return _fac_cache[case]


@pytest.mark.parametrize("case", ["cov2d_1024", "laplace3d_4096", "osc2d_4096"])
def test_matvec_matches_oracle(case):
    _, _, _, h2, _ = problem(case)
    rng = np.random.default_rng(1)
    x = rng.standard_normal(h2.n)
    with one_thread():
        ref = O.matvec(h2, x)
    y = H.matvec(h2, x)
    assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)
    X = rng.standard_normal((h2.n, 3))
    Y = H.matvec(h2, X)
    for j in range(3):
        with one_thread():
            r = O.matvec(h2, X[:, j])
        assert np.linalg.norm(Y[:, j] - r) <= 1e-13 * np.linalg.norm(r)


@pytest.mark.parametrize("case", ROBUST + SENSITIVE)
def test_norm_estimate(case):
    g = load(case)
    _, _, _, h2, _ = problem(case)
    est = H.estimate_norm2(h2)
    assert abs(est - float(g["norm_estimate"])) <= 1e-12 * float(g["norm_estimate"])


@pytest.mark.parametrize("case", ROBUST)
def test_structure_bit_exact(case):
    g = load(case)
    h2, prm, fac = gpu_factor(case)
    assert structure_of(fac) == golden_structure(g)
    for lv, rec in zip(g["levels"], fac.records):
        assert np.array_equal(rec.up_index, g[f"up_index_{lv['level']}"])
        assert {str(c): o for c, o in rec.offset.items()} == lv["offset"]
        for c, f in rec.factors.items():
            assert [[o, k, list(m.shape)] for o, k, m in f.edges] == lv["edges"][str(c)]
    assert fac.top_size == int(g["top_size"])
    assert fac.nbytes() == int(g["factor_bytes"])


@pytest.mark.parametrize("case", ROBUST)
def test_fill_keys_after_every_batch_match_reference(case):
    # golden `fills`: sorted F-key set after each batch (make_golden.py elim_spy)
    g = load(case)
    _, _, fac = gpu_factor(case)
    got = []
    for rec in fac.records:
        got += [[list(k) for k in ks] for ks in rec.fill_keys_after_batches()]
    assert got == g["fills"]


@pytest.mark.parametrize("case", ROBUST)
def test_pivots_match_reference(case, monkeypatch):
    """LU pivots depend on the redundant columns of Q~, which are not unique
    (any orthonormal completion of b_aug).  With the
    reference's construction -- a complete Householder QR of b_aug,
    H2F_COMPLEMENT_QR=1 -- every pivot sequence equals the reference's; the
    default completion (V_perp U_rest from the Jacobi) is checked by
    test_default_completion_pivots_and_solution."""
    g = load(case)
    _, _, _, h2, prm = problem(case)
    monkeypatch.setenv("H2F_COMPLEMENT_QR", "1")
    fac = H.factorize(h2, prm["eps_lu"])
    monkeypatch.delenv("H2F_COMPLEMENT_QR")
    mism, total = 0, 0
    for lv, rec in zip(g["levels"], fac.records):
        for c, f in rec.factors.items():
            want = lv["piv"][str(c)]
            got = None if f.piv is None else f.piv.tolist()
            total += 1
            mism += got != want
    assert np.array_equal(fac.top_piv.astype(np.int64), g["top_piv"])
    # rounding-level differences of the SVD (Jacobi vs dgesdd) can still move
    # one partial-pivoting choice among hundreds of clusters (configs[0]: 1 of 504)
    assert mism <= total // 400, f"{mism} of {total} clusters pivot differently"


@pytest.mark.parametrize("case", ROBUST)
def test_default_completion_pivots_and_solution(case):
    """Default Q~ completion: the integer structure is the reference's (see
    test_structure_bit_exact); pivot sequences may differ where the
    redundant rotation moves a partial-pivoting choice (measured: 5 of 504
    clusters at configs[0]), the solution stays the reference's to 1e-8."""
    g = load(case)
    h2, prm, fac = gpu_factor(case)
    mism, total = 0, 0
    for lv, rec in zip(g["levels"], fac.records):
        for c, f in rec.factors.items():
            total += 1
            mism += (None if f.piv is None else f.piv.tolist()) != lv["piv"][str(c)]
    assert mism <= max(1, total // 50), f"{mism} of {total}"
    b = rhs(h2, H.matvec)
    x = H.refined_solve(h2, fac, b, steps=1)
    assert np.linalg.norm(x - g["x"]) <= 1e-8 * np.linalg.norm(g["x"])


@pytest.mark.parametrize("case", ROBUST + [c for c in SENSITIVE if c not in CHAOTIC])
def test_solution_and_backward_error(case):
    g = load(case)
    h2, prm, fac = gpu_factor(case)
    b = rhs(h2, H.matvec)
    x = H.refined_solve(h2, fac, b, steps=1)
    raw = H.solve(fac, b)

    def eb(v):
        return np.linalg.norm(H.matvec(h2, v) - b) / np.linalg.norm(b)

    assert eb(x) <= 10 * max(float(g["e_b"]), 1e-15)
    assert eb(raw) <= 10 * max(float(g["e_b_raw"]), 1e-15)
    if case in ROBUST:
        assert np.linalg.norm(x - g["x"]) <= 1e-8 * np.linalg.norm(g["x"])


@pytest.mark.parametrize("case", ["cov2d_1024", "cov3d_2048"])
def test_skeleton_projectors_match_oracle(case):
    h2, prm, fac = gpu_factor(case)
    with one_thread():
        ofac = O.factorize(h2, prm["eps_lu"])
    # only the leaf level shares a coordinate system between implementations:
    # above it, each side works in its own (rotation-equivalent) skeleton
    # coordinates of the children
    worst = 0.0
    for rec, orec in zip(fac.records, ofac.records):
        for c, f in rec.factors.items():
            assert f.r == orec.factors[c].r
    rec, orec = fac.records[0], ofac.records[0]
    for c, f in rec.factors.items():
        of = orec.factors[c]
        qs, oqs = f.q[:, f.r:], of.q[:, of.r:]
        worst = max(worst, np.abs(qs @ qs.T - oqs @ oqs.T).max())
    assert worst <= 1e-10, worst


@pytest.mark.parametrize("case", ["cov2d_1024", "laplace2d_2048"])
def test_rotations_orthogonal(case):
    _, _, fac = gpu_factor(case)
    for rec in fac.records:
        for f in rec.factors.values():
            dim = f.q.shape[0]
            assert np.abs(f.q.T @ f.q - np.eye(dim)).max() <= 1e-12 * dim


def test_solve_linear_multi_and_deterministic():
    h2, prm, fac = gpu_factor("cov2d_1024")
    rng = np.random.default_rng(3)
    b1, b2 = rng.standard_normal(fac.n), rng.standard_normal(fac.n)
    lhs = H.solve(fac, 0.7 * b1 - 2.3 * b2)
    rhs_ = 0.7 * H.solve(fac, b1) - 2.3 * H.solve(fac, b2)
    assert np.linalg.norm(lhs - rhs_) <= 1e-10 * np.linalg.norm(lhs)
    B = rng.standard_normal((fac.n, 5))
    X = H.solve_multi(fac, B)
    for j in range(5):
        one = H.solve(fac, B[:, j])
        assert np.linalg.norm(X[:, j] - one) <= 1e-12 * np.linalg.norm(one)
    assert np.array_equal(H.solve(fac, b1), H.solve(fac, b1))
    assert np.array_equal(X, H.solve_multi(fac, B, threads=4))


def test_solve_validates_shapes():
    _, _, fac = gpu_factor("cov2d_1024")
    with pytest.raises(ValueError):
        H.solve(fac, np.zeros(fac.n + 1))
    with pytest.raises(ValueError):
        H.solve_multi(fac, np.zeros(fac.n))
    with pytest.raises(ValueError):
        H.solve_multi(fac, np.zeros((fac.n + 2, 3)))


def test_factor_oracle_oracle_agreement_on_solution():
    # the oracle is the checker: same input, raw solutions agree closely
    h2, prm, fac = gpu_factor("cov3d_2048")
    with one_thread():
        ofac = O.factorize(h2, prm["eps_lu"])
        b = rhs(h2, O.matvec)
        xo = O.substitute(ofac, b)
    xg = H.solve(fac, b)
    assert np.linalg.norm(xg - xo) <= 1e-8 * np.linalg.norm(xo)


def test_singular_leaf_block_names_cluster():
    _, _, _, h2, prm = problem("cov2d_1024")
    leaf = int(h2.tree.levels[h2.tree.depth][0])
    import copy
    bad = copy.copy(h2)
    bad.dense = dict(h2.dense)
    bad.dense[(leaf, leaf)] = np.zeros_like(h2.dense[(leaf, leaf)])
    with pytest.raises(H.FactorizationError, match="cluster"):
        H.factorize(bad, 1e-6)


def test_factorize_bitwise_deterministic():
    _, _, _, h2, prm = problem("cov2d_1024")
    f1 = H.factorize(h2, prm["eps_lu"])
    f2 = H.factorize(h2, prm["eps_lu"], threads=4)
    b = np.random.default_rng(8).standard_normal(h2.n)
    assert np.array_equal(H.solve(f1, b), H.solve(f2, b))
    r1, r2 = f1.records[0], f2.records[0]
    c = r1.clusters[0]
    assert np.array_equal(r1.factors[c].q, r2.factors[c].q)


@pytest.mark.parametrize("case", ["cov2d_4096", "cov3d_2048", "laplace3d_4096"])
def test_large_n_path_matches_shared_memory_path(case, monkeypatch):
    """Force the blocked-Householder QR + multi-CTA Jacobi (used for n > 144
    at upper levels of large problems) on small inputs and compare with the
    shared-memory path: same integer structure, same solution."""
    g = load(case)
    _, _, _, h2, prm = problem(case)
    monkeypatch.setenv("H2F_SMALL_N_MAX", "8")
    fac_big = H.factorize(h2, prm["eps_lu"])
    monkeypatch.delenv("H2F_SMALL_N_MAX")
    _, _, fac = gpu_factor(case)
    assert structure_of(fac_big) == structure_of(fac)
    b = rhs(h2, H.matvec)
    x1 = H.refined_solve(h2, fac_big, b)
    x2 = H.refined_solve(h2, fac, b)
    assert np.linalg.norm(x1 - x2) <= 1e-8 * np.linalg.norm(x2)
    if case != "laplace3d_4096":
        assert structure_of(fac_big) == golden_structure(g)


@pytest.mark.parametrize("case", ["cov2d_4096", "cov3d_2048"])
def test_householder_complement_path_matches_jacobi_completion(case, monkeypatch):
    """Q~'s leading columns come from the Jacobi's complete U (V_perp U_rest)
    by default and from a second complete Householder QR as the fallback
    (H2F_COMPLEMENT_QR=1, also used for numerically rank-deficient fill):
    both are orthonormal completions, the structure is the reference's and
    the solutions agree to the factor tolerance."""
    g = load(case)
    _, _, _, h2, prm = problem(case)
    monkeypatch.setenv("H2F_COMPLEMENT_QR", "1")
    fac_q = H.factorize(h2, prm["eps_lu"])
    monkeypatch.delenv("H2F_COMPLEMENT_QR")
    _, _, fac = gpu_factor(case)
    assert structure_of(fac_q) == golden_structure(g) == structure_of(fac)
    for rec in fac_q.records[:2]:
        for f in rec.factors.values():
            assert np.abs(f.q.T @ f.q - np.eye(f.q.shape[0])).max() <= 1e-12 * f.q.shape[0]
    b = rhs(h2, H.matvec)
    x1 = H.refined_solve(h2, fac_q, b)
    x2 = H.refined_solve(h2, fac, b)
    assert np.linalg.norm(x1 - x2) <= 1e-8 * np.linalg.norm(x2)


@pytest.mark.parametrize("case", ["cov2d_4096", "cov3d_2048"])
def test_blocked_lu_and_dmma_trsm_paths(case, monkeypatch):
    """Force the large-r elimination kernels (cooperative-panel LU, blocked
    DMMA TRSM; used for r > 192 / r >= 48) onto every cluster: pivots and the
    whole integer structure stay bit-exact with the reference golden
    fixture, the solution within 1e-8 of the default path."""
    g = load(case)
    _, _, _, h2, prm = problem(case)
    monkeypatch.setenv("H2F_LU_BLOCKED_MIN", "0")
    monkeypatch.setenv("H2F_TRSM_DMMA_MIN", "1")
    monkeypatch.setenv("H2F_COMPLEMENT_QR", "1")  # the reference's Q~ construction: pivots comparable
    fac_b = H.factorize(h2, prm["eps_lu"])
    monkeypatch.delenv("H2F_LU_BLOCKED_MIN")
    monkeypatch.delenv("H2F_TRSM_DMMA_MIN")
    monkeypatch.delenv("H2F_COMPLEMENT_QR")
    _, _, fac = gpu_factor(case)
    assert structure_of(fac_b) == golden_structure(g)
    for lv, rec in zip(g["levels"], fac_b.records):
        for c, f in rec.factors.items():
            assert (None if f.piv is None else f.piv.tolist()) == lv["piv"][str(c)]
    b = rhs(h2, H.matvec)
    x1 = H.refined_solve(h2, fac_b, b)
    x2 = H.refined_solve(h2, fac, b)
    assert np.linalg.norm(x1 - x2) <= 1e-8 * np.linalg.norm(x2)


def test_solve_multi_sharded_single_rank():
    """The column-sharded multi-RHS path (config 5) on one GPU: without a
    process group it is solve_multi; inside a world-size-1 NCCL group the
    all-gather runs on the device and returns the same bits."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_2509_11152_b200.multigpu import solve_multi_sharded

    h2, prm, fac = gpu_factor("cov2d_1024")
    B = np.random.default_rng(21).standard_normal((fac.n, 7))
    X = H.solve_multi(fac, B)
    assert np.array_equal(solve_multi_sharded(fac, B), X)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        assert np.array_equal(solve_multi_sharded(fac, B), X)
        with pytest.raises(ValueError):
            solve_multi_sharded(fac, B[:-1])
    finally:
        dist.destroy_process_group()
    for j in [0, 6]:
        one = H.solve(fac, B[:, j])
        assert np.linalg.norm(X[:, j] - one) <= 1e-12 * np.linalg.norm(one)


@pytest.mark.parametrize("case,q", [("cov2d_4096", 16), ("laplace3d_4096", 40)])
def test_solve_multi_block_path_matches_single_vector_path(case, q):
    """nrhs >= 4 runs the block substitution (DMMA GEMM rotations/products/
    gathers, DMMA TRSM, blocked top solve); every column must agree with the
    single-vector kernels and with the oracle's substitution."""
    h2, prm, fac = gpu_factor(case)
    B = np.random.default_rng(5).standard_normal((fac.n, q))
    X = H.solve_multi(fac, B)
    for j in [0, q // 2, q - 1]:
        one = H.solve(fac, B[:, j])
        assert np.linalg.norm(X[:, j] - one) <= 1e-11 * np.linalg.norm(one)
    with one_thread():
        of = O.factorize(h2, prm["eps_lu"])
        Xo = O.substitute(of, B[:, :3])
    if case.startswith("cov2d"):
        assert np.linalg.norm(X[:, :3] - Xo) <= 1e-8 * np.linalg.norm(Xo)


def test_device_harness_report_matches_reference_schema():
    """The device harness (reference harness.run, harness.py:197-249) returns
    the reference report keys; e_b and the digest follow the GPU path."""
    from paper_2509_11152_b200.harness import ExperimentConfig, run

    rep = run(ExperimentConfig.from_problem("cov2d", 1024))
    for key in ["version", "config", "n", "e_b", "solution_digest", "h2_bytes", "factor_bytes",
                "kmax_construction", "kmax_factorization", "csp_max", "timings", "phases", "levels", "ranks"]:
        assert key in rep
    assert rep["n"] == 1024 and rep["e_b"] <= 1e-10
    assert set(["factorization", "solve"]) <= set(rep["timings"])
    assert "partial_lu" in rep["phases"] and len(rep["levels"]) == len(rep["ranks"])


def _perturbed(h2, seed, p=1e-14):
    # the oracle draws' operator (scripts/oracle_big.py perturb=1e-14 seed=s):
    # dense blocks * (1 + p z), z ~ N(0,1) per block in sorted key order,
    # symmetrised on diagonal blocks
    import copy

    out = copy.copy(h2)
    object.__setattr__(out, "_h2f_device", None)
    if seed == 0:
        return out
    rng = np.random.default_rng(seed)
    dense = {}
    for key in sorted(h2.dense):
        blk = h2.dense[key]
        z = rng.standard_normal(blk.shape)
        if key[0] == key[1]:
            z = 0.5 * (z + z.T)
        dense[key] = blk * (1.0 + p * z)
    out.dense = dense
    return out


@pytest.mark.parametrize("case", CHAOTIC)
def test_backward_error_distribution_chaotic(case):
    # paired draws: the unperturbed operator and 23 rounding-level
    # perturbations, factored + solved on the GPU; the reference algorithm's
    # e_b on the same 24 operators is committed (tests/golden/<case>_draws.json,
    # the oracle pinned to the reference).  Contract: the median refined e_b
    # within 10x of the reference's median, and the two samples not
    # distinguishable (rank-sum test, p > 0.01)
    import json
    import os

    from scipy.stats import mannwhitneyu

    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", f"{case}_draws.json")))
    seeds = [d["seed"] for d in ref["draws"]]
    ref_eb = np.array([d["e_b"] for d in ref["draws"]])
    _, _, _, h2, prm = problem(case)
    x_true = np.random.Generator(np.random.Philox(7)).standard_normal(h2.n)
    got = []
    for sd in seeds:
        hp = _perturbed(h2, sd)
        b = H.matvec(hp, x_true)
        fac = H.factorize(hp, prm["eps_lu"])
        x = H.refined_solve(hp, fac, b, steps=1)
        got.append(np.linalg.norm(H.matvec(hp, x) - b) / np.linalg.norm(b))
        del fac, hp
    got = np.array(got)
    assert np.median(got) <= 10 * np.median(ref_eb), (np.median(got), np.median(ref_eb))
    assert mannwhitneyu(np.log(got), np.log(ref_eb)).pvalue > 0.01
