"""GPU tests of the boundary's contracts beyond the numerics: structure replay
(the oracle's threshold decisions forced onto the device path), concurrent
callers (concurrent solves are safe), device-pointer checks of
the *_dev entry points."""
import ctypes as C
import threading

import numpy as np
import pytest

import paper_2509_11152_b200 as H
from paper_2509_11152_b200 import _lib as L
from golden_util import one_thread, problem, rhs, structure_of
from oracle import h2_oracle as O

pytestmark = pytest.mark.gpu


def oracle_decisions(h2, eps_lu):
    """Run the oracle with its decision recorder on; returns (factor, kept
    rows, created rows)."""
    O.DECISIONS = {}
    try:
        with one_thread():
            ofac = O.factorize(h2, eps_lu)
        d = O.DECISIONS
    finally:
        O.DECISIONS = None
    kept = np.array([r[:3] for r in d.get("kept", [])], dtype=np.int64).reshape(-1, 3)
    made = np.array(d.get("created", []), dtype=np.int64).reshape(-1, 4)
    return ofac, kept, made


@pytest.mark.parametrize("case", ["laplace3d_4096", "osc2d_4096", "laplace2d_2048", "cov2d_1024"])
def test_replay_reproduces_oracle_structure(case):
    """With the oracle's kept counts and fill decisions forced, the device
    path's batches, ranks and sizes equal the oracle's on every level --
    including the families whose own decisions are rounding-sensitive -- and
    the solution then agrees with the oracle's to the factor tolerance."""
    _, _, _, h2, prm = problem(case)
    ofac, kept, made = oracle_decisions(h2, prm["eps_lu"])
    L.replay_set(kept, made)
    try:
        fac = H.factorize(h2, prm["eps_lu"])
        stats = L.replay_stats()
    finally:
        L.replay_clear()
    assert stats["kept_forced"] > 0
    assert structure_of(fac) == structure_of(ofac)
    assert fac.top_size == ofac.top_size
    for rec in fac.records:
        _, events = rec.fill_events()
        want = sorted((int(a), int(b)) for lv, _, a, b in made if lv == rec.level)
        assert sorted(k for _, k in events) == want
    b = rhs(h2, H.matvec)
    with one_thread():
        xo = O.substitute(ofac, b)
    xg = H.solve(fac, b)
    assert np.linalg.norm(xg - xo) <= 1e-6 * np.linalg.norm(xo)


def test_replay_cleared_restores_own_decisions():
    _, _, _, h2, prm = problem("laplace3d_4096")
    f1 = H.factorize(h2, prm["eps_lu"])
    _, kept, made = oracle_decisions(h2, prm["eps_lu"])
    # the oracle's fill but no kept counts: the first cluster with fill to
    # augment has no replayed decision
    L.replay_set(np.zeros((0, 3), np.int64), made)
    try:
        with pytest.raises(ValueError, match="replay"):
            H.factorize(h2, prm["eps_lu"])
    finally:
        L.replay_clear()
    f2 = H.factorize(h2, prm["eps_lu"])
    assert structure_of(f1) == structure_of(f2)


def test_concurrent_solves_match_serial():
    """ctypes releases the GIL: four threads solving on one factor at once
    must give the serial bits (the library serialises its entry points)."""
    _, _, _, h2, prm = problem("cov2d_4096")
    fac = H.factorize(h2, prm["eps_lu"])
    rng = np.random.default_rng(3)
    bs = [rng.standard_normal(fac.n) for _ in range(4)]
    Bm = rng.standard_normal((fac.n, 6))
    want = [H.solve(fac, b) for b in bs]
    want_m = H.solve_multi(fac, Bm)
    want_r = H.refined_solve(h2, fac, bs[0])
    got, errs = {}, []

    def work(i):
        try:
            for rep in range(3):
                got[(i, rep)] = H.solve(fac, bs[i])
                if i == 0:
                    got[("m", rep)] = H.solve_multi(fac, Bm)
                if i == 1:
                    got[("r", rep)] = H.refined_solve(h2, fac, bs[0])
        except Exception as exc:  # pragma: no cover - reported below
            errs.append(exc)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for i in range(4):
        for rep in range(3):
            assert np.array_equal(got[(i, rep)], want[i])
    for rep in range(3):
        assert np.array_equal(got[("m", rep)], want_m)
        assert np.array_equal(got[("r", rep)], want_r)


def test_dev_entry_points_reject_host_pointers():
    _, _, _, h2, prm = problem("cov2d_1024")
    fac = H.factorize(h2, prm["eps_lu"])
    b = np.ones(fac.n)
    x = np.zeros(fac.n)
    lib = L.ensure_init()
    code = lib.h2f_solve_dev(fac._h.ptr, C.c_void_p(b.ctypes.data), C.c_void_p(x.ctypes.data), 1)
    assert code == L.H2F_E_ARG
    assert "host pointer" in L.last_error() or "not a CUDA pointer" in L.last_error()
    # the context is still usable afterwards
    assert np.all(np.isfinite(H.solve(fac, b)))


def test_refined_solve_multi_matches_columns():
    """Block refinement: every column equals the
    single-vector refined_solve up to rounding, and the backward error of
    each column is at the refined level."""
    _, _, _, h2, prm = problem("cov2d_4096")
    fac = H.factorize(h2, prm["eps_lu"])
    B = np.random.default_rng(11).standard_normal((fac.n, 6))
    X = H.refined_solve_multi(h2, fac, B, steps=1)
    for j in range(6):
        xj = H.refined_solve(h2, fac, B[:, j], steps=1)
        assert np.linalg.norm(X[:, j] - xj) <= 1e-12 * np.linalg.norm(xj)
    R = H.matvec(h2, X) - B
    assert np.linalg.norm(R) <= 1e-9 * np.linalg.norm(B)
    with pytest.raises(ValueError):
        H.refined_solve_multi(h2, fac, B[:-1])


def test_factor_save_load_round_trip(tmp_path):
    """f2: a saved and re-imported factor solves bit for bit like the
    original; records, batches, ranks, pivots and nbytes survive."""
    _, _, _, h2, prm = problem("laplace3d_4096")
    fac = H.factorize(h2, prm["eps_lu"])
    path = tmp_path / "fac.npz"
    H.save_factorization(fac, path)
    fac2 = H.load_factorization(path, h2.tree)
    assert fac2.nbytes() == fac.nbytes() and fac2.top_size == fac.top_size
    assert structure_of(fac2) == structure_of(fac)
    b = np.random.default_rng(2).standard_normal(fac.n)
    assert np.array_equal(H.solve(fac2, b), H.solve(fac, b))
    B = np.random.default_rng(3).standard_normal((fac.n, 5))
    assert np.array_equal(H.solve_multi(fac2, B), H.solve_multi(fac, B))
    assert np.array_equal(H.refined_solve(h2, fac2, b), H.refined_solve(h2, fac, b))
    c = fac.records[0].clusters[3]
    assert np.array_equal(fac2.records[0].factors[c].piv, fac.records[0].factors[c].piv)
    with pytest.raises(ValueError):
        from paper_2509_11152_b200.serialize import unpack
        unpack({"meta": np.array('{"format": "other"}')})


def test_solve_plans_bounded_for_many_column_counts():
    """a solve plan per nrhs used to stay cached forever; the
    cache is now LRU-bounded, so ragged column counts do not grow the arena."""
    _, _, _, h2, prm = problem("cov2d_1024")
    fac = H.factorize(h2, prm["eps_lu"])
    rng = np.random.default_rng(9)
    in_use = {}
    for q in range(5, 41):
        B = rng.standard_normal((fac.n, q))
        X = H.solve_multi(fac, B)
        # raw substitution: residual at the factorization tolerance (~1e-7 here)
        assert np.linalg.norm(H.matvec(h2, X) - B) <= 1e-5 * np.linalg.norm(B)
        in_use[q] = L.memory_stats()["in_use"]
    # 28 more distinct column counts after q = 12: bounded by the 3 live plans
    per_plan = max(in_use[8] - in_use[7], 1)
    assert in_use[40] - in_use[12] <= 3 * per_plan + (64 << 20), (in_use[12], in_use[40], per_plan)


def test_solve_graph_replay_same_bits_and_launch_count():
    """The single-vector substitution is captured into a CUDA graph on first
    use and replayed; with the per-kernel profiler on it runs launch by launch.
    Same bits either way, and the launch counter counts the replayed kernels."""
    _, _, _, h2, prm = problem("laplace3d_4096")
    fac = H.factorize(h2, prm["eps_lu"])
    b = np.random.default_rng(12).standard_normal(fac.n)
    x0 = H.solve(fac, b)              # direct (uses 1, 2)
    assert np.array_equal(x0, H.solve(fac, b))
    x1 = H.solve(fac, b)              # third use: captured
    c0 = L.kernel_launches()
    x2 = H.solve(fac, b)              # replays
    replayed = L.kernel_launches() - c0
    L.profile_enable(True)
    try:
        c0 = L.kernel_launches()
        x3 = H.solve(fac, b)          # launch by launch
        direct = L.kernel_launches() - c0
    finally:
        L.profile_enable(False)
    assert np.array_equal(x1, x2) and np.array_equal(x1, x3) and np.array_equal(x0, x1)
    assert replayed == direct > 0
