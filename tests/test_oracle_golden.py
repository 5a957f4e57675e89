"""Pin the CPU oracle (oracle/h2_oracle.py) and the problem builder
(paper_2509_11152_b200/problem.py) against fixtures produced by the
reference itself (tests/golden/make_golden.py)."""
import hashlib

import numpy as np
import pytest

from golden_util import CASES, golden_structure, h2_digest, load, one_thread, problem, rhs, structure_of
from oracle import h2_oracle as O

FAST = ["cov2d_1024", "cov3d_2048", "laplace2d_2048", "helmholtz3d_2048"]
SLOW = ["cov2d_4096", "laplace3d_4096", "osc2d_4096", "cov3d_e8_4096", "cov2d_16384", "lru_cov3d_4096"]


@pytest.mark.parametrize("case", list(CASES))
def test_builder_matches_reference_input(case):
    g = load(case)
    _, _, _, h2, _ = problem(case)
    assert h2_digest(h2) == str(g["h2_digest"])


@pytest.mark.parametrize("case", FAST + SLOW)
def test_oracle_reproduces_reference(case):
    g = load(case)
    _, _, _, h2, prm = problem(case)
    with one_thread():
        fac = O.factorize(h2, prm["eps_lu"])
        b = rhs(h2, O.matvec)
        x = O.refined_solve(h2, fac, b, steps=1)
    assert fac.norm_estimate == float(g["norm_estimate"])
    assert fac.eps_fill == float(g["eps_fill"])
    assert structure_of(fac) == golden_structure(g)
    for lv, rec in zip(g["levels"], fac.records):
        assert np.array_equal(rec.up_index, g[f"up_index_{lv['level']}"])
        for c, f in rec.factors.items():
            assert [[int(o), k, list(m.shape)] for o, k, m in f.edges] == lv["edges"][str(c)]
            want = lv["piv"][str(c)]
            assert (None if f.piv is None else f.piv.tolist()) == want
    assert fac.top_size == int(g["top_size"])
    assert np.array_equal(fac.top_piv.astype(np.int64), g["top_piv"])
    assert fac.nbytes() == int(g["factor_bytes"])
    # bitwise: same LAPACK calls in the same order, one BLAS thread
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(g["x_digest"])
