"""Substitution against a B200 factorization (solve.py:29-77 of the reference).

solve(fac, b), solve_multi(fac, B), refined_solve(h2, fac, b, steps) keep the
reference's signatures, shape checks and ValueError messages; `threads` is
accepted for API parity.
"""
from __future__ import annotations

import numpy as np

from . import _lib as L
from .h2core import device_matrix

__all__ = ["solve", "solve_multi", "refined_solve", "refined_solve_multi"]


def solve(fac, b, threads=1):
    """x with (factored matrix) x = b, both in tree order."""
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (fac.n,):
        raise ValueError(f"right-hand side must have shape ({fac.n},)")
    return _run(fac, b, 1)


def solve_multi(fac, b, threads=1):
    """Block variant of solve for an n x q right-hand side."""
    b = np.asarray(b, dtype=np.float64)
    if b.ndim != 2 or b.shape[0] != fac.n:
        raise ValueError(f"right-hand side must have shape ({fac.n}, q)")
    return _run(fac, b, b.shape[1])


def _run(fac, b, nrhs):
    bc = np.ascontiguousarray(b)
    x = np.empty_like(bc)
    if bc.size:
        L.check(L.lib().h2f_solve(fac.handle.ptr, L.ptr(bc), L.ptr(x), nrhs), "h2f_solve")
    return x


def refined_solve(h2, fac, b, threads=1, steps=1):
    """Substitution followed by `steps` rounds of iterative refinement
    against h2 (one matvec + one substitution each)."""
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (fac.n,):
        raise ValueError(f"right-hand side must have shape ({fac.n},)")
    dev = device_matrix(h2)
    bc = np.ascontiguousarray(b)
    x = np.empty_like(bc)
    L.check(L.lib().h2f_refined_solve(dev.handle, fac.handle.ptr, L.ptr(bc), L.ptr(x), int(steps)),
            "h2f_refined_solve")
    return x


def refined_solve_multi(h2, fac, b, threads=1, steps=1):
    """refined_solve for an n x q block of right-hand sides: block
    substitution, then `steps` rounds of (block matvec, block substitution).
    Column j equals refined_solve(h2, fac, b[:, j]) up to rounding
    (extension of solve.py:63-77)."""
    b = np.asarray(b, dtype=np.float64)
    if b.ndim != 2 or b.shape[0] != fac.n:
        raise ValueError(f"right-hand side must have shape ({fac.n}, q)")
    dev = device_matrix(h2)
    bc = np.ascontiguousarray(b)
    x = np.empty_like(bc)
    if bc.size:
        L.check(L.lib().h2f_refined_solve_multi(dev.handle, fac.handle.ptr, L.ptr(bc), L.ptr(x), b.shape[1],
                                                int(steps)), "h2f_refined_solve_multi")
    return x
