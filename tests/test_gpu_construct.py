"""Device H2 construction (h2core.py:128-269 build_h2 +
orthogonalize_recompress) against the host builder, which is the reference's
construction restated bit-for-bit (digest-tested in test_oracle_golden.py).

Contract (tolerance -- GPU exp/cos/log and batched QR/SVD round
differently from NumPy/LAPACK):
  * ranks: identical per cluster (integer structure),
  * operator: |A_dev x - A_host x| <= 1e-8 |A_host x|,
  * approximation: dense-kernel error of the device operator within 1% of
    the host operator's,
  * downstream: factor + refined solve on the device operator within 10x of
    the host operator's backward error.
"""
import numpy as np
import pytest

import paper_2509_11152_b200 as H
from paper_2509_11152_b200 import problem as P
from paper_2509_11152_b200.construct import build_h2_device, build_problem_device, export_blocks

pytestmark = pytest.mark.gpu

CASES = {
    "cov2d_4096": ("cov2d", 4096, {}),
    "laplace3d_4096": ("helmholtz3d", 4096, {"kappa": 0.0}),
    "osc2d_4096": ("helmholtz3d", 4096, {"dim": 2, "p0": 8, "eta": 0.9}),
    "laplace2d_2048": ("laplace2d", 2048, {}),
    "cov3d_e8_4096": ("cov3d", 4096, {"eps_lu": 1e-8}),
    # + the seeded rank-32 update absorbed on the device (h2core.py:342-405)
    "lru_cov3d_4096": ("lru_cov3d", 4096, {}),
}
_cache = {}


def both(case):
    if case not in _cache:
        name, n, over = CASES[case]
        _, _, _, hh, prm = P.build_problem(name, n, **over)
        tree, part, spec, hd, _ = build_problem_device(name, n, **over)
        _cache[case] = (hh, hd, spec, prm)
    return _cache[case]


def ranks(h2):
    return np.array([h2.rank.get(c, -1) for c in range(len(h2.tree.parent))])


@pytest.mark.parametrize("case", sorted(CASES))
def test_ranks_and_operator_match_host_builder(case):
    hh, hd, spec, prm = both(case)
    assert np.array_equal(ranks(hd), ranks(hh))
    x = np.random.default_rng(1).standard_normal(hh.n)
    yh, yd = H.matvec(hh, x), H.matvec(hd, x)
    assert np.linalg.norm(yd - yh) <= 1e-8 * np.linalg.norm(yh)
    rows = np.random.default_rng(2).choice(hh.n, size=128, replace=False)
    ex = P.entry_block(spec, hh.tree.points, rows, np.arange(hh.n)) @ x
    if prm.get("lru_rank", 0):
        w = P.make_low_rank_factor(hh.n, prm["lru_rank"], prm.get("seed", 7))
        ex = ex + w[rows] @ (w.T @ x)
    err_h = np.linalg.norm(yh[rows] - ex) / np.linalg.norm(ex)
    err_d = np.linalg.norm(yd[rows] - ex) / np.linalg.norm(ex)
    assert err_d <= 1.01 * err_h + 1e-14


@pytest.mark.parametrize("case", sorted(CASES))
def test_factorization_of_device_operator(case):
    hh, hd, spec, prm = both(case)
    xr = P.rhs_for(hh)

    def eb(h2):
        b = H.matvec(h2, xr)
        fac = H.factorize(h2, prm["eps_lu"])
        x = H.refined_solve(h2, fac, b, steps=1)
        return np.linalg.norm(H.matvec(h2, x) - b) / np.linalg.norm(b)

    assert eb(hd) <= 10 * max(eb(hh), 1e-15)


def test_dense_blocks_and_bases_close_to_host():
    hh, hd, spec, prm = both("cov2d_4096")
    blk = export_blocks(hd)
    assert set(blk["dense"]) == set(hh.dense) and set(blk["coupling"]) == set(hh.coupling)
    worst = max(np.abs(blk["dense"][k] - hh.dense[k]).max() / np.abs(hh.dense[k]).max() for k in hh.dense)
    assert worst <= 1e-14
    # bases: orthonormal, spanning the host basis's subspace (columns of
    # near-degenerate singular values are only determined up to rotation)
    for c, v in hh.leaf_basis.items():
        u = blk["leaf_basis"][c]
        assert np.abs(u.T @ u - np.eye(u.shape[1])).max() <= 1e-12
        cos = np.linalg.svd(u.T @ v, compute_uv=False)
        assert cos.min() >= 1 - 1e-3, c


def test_export_round_trip_bitwise():
    hh, hd, spec, prm = both("laplace3d_4096")
    blk = export_blocks(hd)
    h2 = P.H2Matrix(tree=hd.tree, partition=hd.partition, leaf_basis=blk["leaf_basis"],
                    transfer=blk["transfer"], coupling=blk["coupling"], dense=blk["dense"],
                    rank=dict(hd.rank))
    x = np.random.default_rng(3).standard_normal(h2.n)
    assert np.array_equal(H.matvec(h2, x), H.matvec(hd, x))
    # the DeviceH2 exposes the same dicts lazily
    assert set(hd.dense) == set(h2.dense)


def test_interpolation_only_operator():
    # eps <= 0: build_h2 without orthogonalize_recompress (ranks = p^d)
    pts, counts = P.generate_uniform_grid(1024, 2)
    tree = P.build_cluster_tree(pts, 64)
    part = P.dual_tree_traversal(tree, 0.9)
    spec = P.KernelSpec(family="exp_covariance", dim=2, corr_length=0.1, diag_value=1.0)
    hd = build_h2_device(tree, part, spec, 8, 0.0)
    hh = P.build_h2(tree, part, spec, 8)
    assert all(hd.rank[c] == hh.rank[c] for c in hh.rank)
    x = np.random.default_rng(4).standard_normal(1024)
    yh, yd = H.matvec(hh, x), H.matvec(hd, x)
    assert np.linalg.norm(yd - yh) <= 1e-12 * np.linalg.norm(yh)


def test_build_rejects_bad_arguments():
    pts, counts = P.generate_uniform_grid(1024, 2)
    tree = P.build_cluster_tree(pts, 64)
    part = P.dual_tree_traversal(tree, 0.9)
    with pytest.raises(ValueError):
        build_h2_device(tree, part, P.KernelSpec(family="nope", dim=2), 8, 1e-6)
    with pytest.raises(ValueError, match="p0"):  # H2F_E_ARG from the library
        build_h2_device(tree, part, P.KernelSpec(family="exp_covariance", dim=2), 0, 1e-6)


def test_harness_and_cli_device_build(tmp_path):
    import json

    from golden_util import load
    from paper_2509_11152_b200 import cli
    from paper_2509_11152_b200.harness import ExperimentConfig, run

    g = load("cov2d_16384")  # configs[0]: construct + factorize + solve
    rep = run(ExperimentConfig.from_problem("cov2d", 16384, device_build=True))
    assert rep["e_b"] <= 10 * float(g["e_b"])
    assert rep["kmax_construction"] == 43 and rep["h2_bytes"] > 0
    assert cli.main(["run", "--problem", "cov2d", "--n", "4096", "--device-build", "--out", str(tmp_path)]) == 0
    assert json.load(open(tmp_path / "report.json"))["config"]["device_build"] is True


def test_absorb_low_rank_on_host_built_operator():
    # device absorb of a host-built operator = host absorb_low_rank (ranks, operator)
    import copy

    _, _, _, h0, prm = P.build_problem("cov3d", 2048)
    w = P.make_low_rank_factor(2048, 16, 3)
    from paper_2509_11152_b200.construct import absorb_low_rank_device

    hh = P.absorb_low_rank(copy.deepcopy(h0), w, prm["eps"])  # (before h0 caches a device handle)
    hd = absorb_low_rank_device(h0, w, prm["eps"])
    assert np.array_equal(ranks(hd), ranks(hh))
    x = np.random.default_rng(5).standard_normal(2048)
    yh = H.matvec(hh, x)
    assert np.linalg.norm(H.matvec(hd, x) - yh) <= 1e-8 * np.linalg.norm(yh)
    # the input operator is untouched
    y0 = H.matvec(h0, x)
    assert np.linalg.norm(y0 - yh) > 1e-6 * np.linalg.norm(yh)
