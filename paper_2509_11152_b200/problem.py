"""Synthetic problem builder: points, KD cluster tree, block partition,
kernel entries and the nested-basis H2 operator that the factorization
consumes.

This is the INPUT side of the hot path ("next" row
f1).  It runs on the host in NumPy/SciPy, exactly like the reference, so
that the operator handed to the B200 factorization is bit-for-bit the one
the reference would factor on the same machine (checked against the
reference in tests/test_oracle_golden.py::test_builder_matches_reference_input).  Nothing here is timed as part
of the path.

Reference behaviour restated (file:line under /root/reference/pkg/src/h2factor):
  grid + tree          geometry.py:26-63, 145-229
  box metrics          geometry.py:66-82
  partition            structure.py:30-124
  kernels              kernels.py:44-106
  Chebyshev bases      h2core.py:39-94
  build_h2             h2core.py:128-174
  recompression        h2core.py:177-269
  low-rank update      h2core.py:333-392 (absorb_low_rank), kernels.py:89-96
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
from scipy.spatial.distance import cdist
from threadpoolctl import threadpool_limits

__all__ = [
    "PROBLEMS",
    "ClusterTree",
    "BlockPartition",
    "KernelSpec",
    "H2Matrix",
    "generate_uniform_grid",
    "build_cluster_tree",
    "dual_tree_traversal",
    "sparsity_constant",
    "default_diag_value",
    "entry_block",
    "eval_kernel",
    "build_h2",
    "orthogonalize_recompress",
    "h2_nbytes",
    "build_problem",
    "rhs_for",
    "make_low_rank_factor",
    "absorb_low_rank",
]

# --------------------------------------------------------------------------
# problem table (harness.py:55-71)
# --------------------------------------------------------------------------

PROBLEMS = {
    "cov2d": dict(family="exp_covariance", dim=2, m=64, p0=8, eta=0.9,
                  alpha_r=1e-2, eps=1e-7, eps_lu=1e-6, corr_length=0.1,
                  kappa=3.0),
    "cov3d": dict(family="exp_covariance", dim=3, m=64, p0=4, eta=0.7,
                  alpha_r=1e-2, eps=1e-7, eps_lu=1e-6, corr_length=0.2,
                  kappa=3.0),
    "laplace2d": dict(family="laplace2d", dim=2, m=64, p0=8, eta=0.9,
                      alpha_r=1e-5, eps=1e-7, eps_lu=1e-6, corr_length=0.1,
                      kappa=3.0),
    "helmholtz3d": dict(family="helmholtz3d", dim=3, m=64, p0=4, eta=0.7,
                        alpha_r=1e-2, eps=1e-7, eps_lu=1e-6, corr_length=0.1,
                        kappa=3.0),
    # 3D covariance with a seeded rank-32 symmetric update W W^T folded into
    # the representation before factorization (harness.py:68-70, 185-189)
    "lru_cov3d": dict(family="exp_covariance", dim=3, m=128, p0=4, eta=0.9,
                      alpha_r=1e-2, eps=1e-8, eps_lu=1e-7, corr_length=0.2,
                      kappa=3.0, lru_rank=32),
}


# --------------------------------------------------------------------------
# points and the cluster tree
# --------------------------------------------------------------------------

def _divisors(n):
    small, large = [], []
    i = 1
    while i * i <= n:
        if n % i == 0:
            small.append(i)
            if i * i != n:
                large.append(n // i)
        i += 1
    return small + large[::-1]


def _ordered_factorizations(n, d):
    """All ordered d-tuples of positive ints with product n."""
    if d == 1:
        return [(n,)]
    out = []
    for a in _divisors(n):
        for rest in _ordered_factorizations(n // a, d - 1):
            out.append((a,) + rest)
    return out


def _grid_counts(n, d):
    # most balanced split (max/min ratio, ties by the lexicographically
    # smallest ordered tuple), reported largest first  (geometry.py:26-48)
    best = min((max(t) / min(t), t) for t in _ordered_factorizations(n, d))
    return tuple(sorted(best[1], reverse=True))


def generate_uniform_grid(n, d):
    """Cell centres of a uniform n-point grid on the unit cube, first axis
    slowest (geometry.py:51-63)."""
    if n <= 0 or d not in (2, 3):
        raise ValueError(f"need n >= 1 and d in (2, 3), got n={n} d={d}")
    counts = _grid_counts(n, d)
    axes = [(np.arange(c) + 0.5) / c for c in counts]
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([g.reshape(-1) for g in mesh], axis=1), counts


def _diag_len(lo, hi):
    return float(np.linalg.norm(np.asarray(hi) - np.asarray(lo)))


def _centre_gap(lo_a, hi_a, lo_b, hi_b):
    ca = (np.asarray(lo_a) + np.asarray(hi_a)) / 2.0
    cb = (np.asarray(lo_b) + np.asarray(hi_b)) / 2.0
    return float(np.linalg.norm(ca - cb))


@dataclass
class ClusterTree:
    """Binary KD tree in preorder; same fields as the reference's
    ClusterTree (geometry.py:85-142) so either can drive factorize()."""

    points: np.ndarray
    perm: np.ndarray
    m_leaf: int
    parent: np.ndarray
    child_left: np.ndarray
    child_right: np.ndarray
    level: np.ndarray
    begin: np.ndarray
    end: np.ndarray
    box_lo: np.ndarray
    box_hi: np.ndarray
    depth: int
    levels: list = field(default_factory=list)

    @property
    def n(self):
        return self.points.shape[0]

    @property
    def dim(self):
        return self.points.shape[1]

    @property
    def num_nodes(self):
        return self.parent.shape[0]

    def is_leaf(self, i):
        return self.child_left[i] < 0

    def size(self, i):
        return int(self.end[i] - self.begin[i])

    def children(self, i):
        return int(self.child_left[i]), int(self.child_right[i])

    def diameter(self, i):
        return _diag_len(self.box_lo[i], self.box_hi[i])

    def to_tree_order(self, x):
        return np.asarray(x)[..., self.perm]

    def to_original_order(self, x):
        out = np.empty_like(np.asarray(x))
        out[..., self.perm] = np.asarray(x)
        return out


def _uniform_depth(n, m):
    # smallest depth whose ceil(n / 2^depth) fits a leaf (geometry.py:145-150)
    k = 0
    while -(-n // (1 << k)) > m and (1 << k) < n:
        k += 1
    return k


def build_cluster_tree(points, m):
    """KD tree splitting the widest box axis at the median (geometry.py:153-229)."""
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[0] == 0:
        raise ValueError("points must be a nonempty (n, d) array")
    if m < 1:
        raise ValueError("leaf size m must be >= 1")
    n = pts.shape[0]
    depth = _uniform_depth(n, m)
    perm = np.arange(n)
    nodes = []  # rows: [parent, left, right, level, begin, end]
    lo_list, hi_list = [], []

    def add(par, lev, b, e, lo, hi):
        nodes.append([par, -1, -1, lev, b, e])
        lo_list.append(lo)
        hi_list.append(hi)
        return len(nodes) - 1

    def split(node):
        _, _, _, lev, b, e = nodes[node]
        if lev >= depth or e - b < 2:
            return
        lo, hi = lo_list[node], hi_list[node]
        axis = int(np.argmax(hi - lo))
        idx = perm[b:e]
        order = np.lexsort((idx, pts[idx, axis]))
        perm[b:e] = idx[order]
        mid = b + (e - b + 1) // 2
        cut = 0.5 * (pts[perm[mid - 1], axis] + pts[perm[mid], axis])
        hi_left = hi.copy()
        hi_left[axis] = cut
        lo_right = lo.copy()
        lo_right[axis] = cut
        # siblings get consecutive ids, then the left subtree is numbered
        left = add(node, lev + 1, b, mid, lo.copy(), hi_left)
        right = add(node, lev + 1, mid, e, lo_right, hi.copy())
        nodes[node][1], nodes[node][2] = left, right
        split(left)
        split(right)

    split(add(-1, 0, 0, n, pts.min(axis=0).copy(), pts.max(axis=0).copy()))
    arr = np.asarray(nodes, dtype=np.int64)
    tree = ClusterTree(
        points=pts[perm].copy(), perm=perm, m_leaf=m,
        parent=arr[:, 0].copy(), child_left=arr[:, 1].copy(),
        child_right=arr[:, 2].copy(), level=arr[:, 3].copy(),
        begin=arr[:, 4].copy(), end=arr[:, 5].copy(),
        box_lo=np.asarray(lo_list), box_hi=np.asarray(hi_list), depth=depth)
    tree.levels = [np.flatnonzero(tree.level == lv) for lv in range(depth + 1)]
    return tree


# --------------------------------------------------------------------------
# block partition (structure.py:30-124) and sparsity constant (127-134)
# --------------------------------------------------------------------------

def _admissible(tree, s, t, eta):
    if s == t:
        return False
    half_sum = 0.5 * (tree.diameter(s) + tree.diameter(t))
    dist = _centre_gap(tree.box_lo[s], tree.box_hi[s],
                       tree.box_lo[t], tree.box_hi[t])
    return dist > 0.0 and half_sum <= eta * dist


@dataclass
class BlockPartition:
    """Per-level canonical (s <= t) pair lists; attribute names match the
    reference's BlockPartition (structure.py:42-85)."""

    eta: float
    admissible_leaves: list
    inadmissible_inner: list
    inadmissible_leaves: list
    top_level: int | None = None

    def __post_init__(self):
        self._adm = [set(p) for p in self.admissible_leaves]
        self._dense = [set(a) | set(b) for a, b in
                       zip(self.inadmissible_inner, self.inadmissible_leaves)]

    def levels(self):
        return range(len(self.admissible_leaves))

    def dense_pairs(self, level):
        return sorted(self._dense[level])

    def coupling_index(self, level):
        index = {}
        for s, t in self.admissible_leaves[level]:
            index.setdefault(s, []).append(((s, t), False))
            index.setdefault(t, []).append(((s, t), True))
        return index

    def is_dense(self, level, s, t):
        return (min(s, t), max(s, t)) in self._dense[level]

    def is_admissible_leaf(self, level, s, t):
        return (min(s, t), max(s, t)) in self._adm[level]


def dual_tree_traversal(tree, eta):
    nlev = tree.depth + 1
    adm = [[] for _ in range(nlev)]
    inner = [[] for _ in range(nlev)]
    leafd = [[] for _ in range(nlev)]
    work = [(0, 0)]
    while work:
        s, t = work.pop()
        lev = int(tree.level[s])
        if _admissible(tree, s, t, eta):
            adm[lev].append((s, t))
        elif tree.is_leaf(s) or tree.is_leaf(t):
            leafd[lev].append((s, t))
        else:
            inner[lev].append((s, t))
            sl, sr = tree.children(s)
            if s == t:
                work.extend([(sl, sl), (sl, sr), (sr, sr)])
            else:
                tl, tr = tree.children(t)
                work.extend([(sl, tl), (sl, tr), (sr, tl), (sr, tr)])
    for rows in (adm, inner, leafd):
        for pairs in rows:
            pairs.sort()
    part = BlockPartition(eta=eta, admissible_leaves=adm,
                          inadmissible_inner=inner, inadmissible_leaves=leafd)
    with_adm = [lv for lv in range(nlev) if adm[lv]]
    part.top_level = min(with_adm) if with_adm else None
    return part


def sparsity_constant(partition, level):
    """Largest number of dense blocks in one block row at `level`."""
    cnt = {}
    for s, t in partition._dense[level]:
        cnt[s] = cnt.get(s, 0) + 1
        if s != t:
            cnt[t] = cnt.get(t, 0) + 1
    return max(cnt.values()) if cnt else 0


# --------------------------------------------------------------------------
# kernels (kernels.py:29-106)
# --------------------------------------------------------------------------

@dataclass
class KernelSpec:
    family: str
    dim: int
    corr_length: float = 0.1
    kappa: float = 3.0
    diag_value: float = 0.0
    alpha_r: float = 0.0


def _kernel_of_r(spec, r):
    fam = spec.family
    if fam == "exp_covariance":
        return np.exp(-r / spec.corr_length)
    if fam == "laplace2d":
        with np.errstate(divide="ignore"):
            return -np.log(r) / (2.0 * np.pi)
    if fam == "helmholtz3d":
        with np.errstate(divide="ignore", invalid="ignore"):
            return np.cos(spec.kappa * r) / r
    raise ValueError(f"unknown kernel family {fam!r}")


def eval_kernel(spec, x, y):
    return _kernel_of_r(spec, cdist(np.atleast_2d(x), np.atleast_2d(y)))


def entry_block(spec, points, rows, cols):
    rows = np.asarray(rows)
    cols = np.asarray(cols)
    vals = _kernel_of_r(spec, cdist(points[rows], points[cols]))
    same = rows[:, None] == cols[None, :]
    if same.any():
        base = 1.0 if spec.family == "exp_covariance" else spec.diag_value
        vals[same] = base + spec.alpha_r
    return vals


def default_diag_value(family, h):
    if family == "laplace2d":
        return max(0.0, -np.log(h) / (2.0 * np.pi))
    if family == "helmholtz3d":
        return 1.0 / h
    return 1.0


# --------------------------------------------------------------------------
# H2 representation (h2core.py:39-269)
# --------------------------------------------------------------------------

def _cheb_points(p, lo, hi):
    k = np.arange(p)
    t = np.cos((2 * k + 1) * np.pi / (2 * p))
    return 0.5 * (t + 1.0) * (hi - lo) + lo


def _cheb_bary(p):
    k = np.arange(p)
    return (-1.0) ** k * np.sin((2 * k + 1) * np.pi / (2 * p))


def chebyshev_grid(box_lo, box_hi, p):
    axes = [_cheb_points(p, lo, hi) for lo, hi in zip(box_lo, box_hi)]
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([g.ravel() for g in mesh], axis=1)


def _lagrange_rows(x, nodes, w):
    diff = x[:, None] - nodes[None, :]
    hit_r, hit_c = np.nonzero(diff == 0.0)
    with np.errstate(divide="ignore", invalid="ignore"):
        q = w[None, :] / diff
        out = q / np.sum(q, axis=1, keepdims=True)
    if hit_r.size:
        out[hit_r] = 0.0
        out[hit_r, hit_c] = 1.0
    return out


def interpolation_matrix(points, box_lo, box_hi, p):
    points = np.asarray(points)
    w = _cheb_bary(p)
    per_axis = [_lagrange_rows(points[:, a], _cheb_points(p, lo, hi), w)
                for a, (lo, hi) in enumerate(zip(box_lo, box_hi))]
    if len(per_axis) == 2:
        out = np.einsum("ia,ib->iab", per_axis[0], per_axis[1])
    else:
        out = np.einsum("ia,ib,ic->iabc", *per_axis)
    return out.reshape(points.shape[0], p ** len(per_axis))


@dataclass
class H2Matrix:
    """Symmetric nested-basis operator; field names match the reference's
    H2Matrix (h2core.py:97-125): dense/coupling hold canonical (s <= t)
    pairs, transfer[c] maps c's coefficients into its parent's."""

    tree: object
    partition: BlockPartition
    leaf_basis: dict = field(default_factory=dict)
    transfer: dict = field(default_factory=dict)
    coupling: dict = field(default_factory=dict)
    dense: dict = field(default_factory=dict)
    rank: dict = field(default_factory=dict)

    @property
    def n(self):
        return self.tree.n


def build_h2(tree, partition, spec, p0):
    h2 = H2Matrix(tree=tree, partition=partition)
    pts = tree.points
    for lv in partition.levels():
        for s, t in partition.inadmissible_leaves[lv]:
            h2.dense[(s, t)] = entry_block(
                spec, pts, np.arange(tree.begin[s], tree.end[s]),
                np.arange(tree.begin[t], tree.end[t]))
    top = partition.top_level
    if top is None:
        return h2
    grid = {}
    for lv in range(tree.depth, top - 1, -1):
        p = p0 + (tree.depth - lv) // 2
        for c in tree.levels[lv]:
            grid[c] = chebyshev_grid(tree.box_lo[c], tree.box_hi[c], p)
            if tree.is_leaf(c):
                h2.leaf_basis[c] = interpolation_matrix(
                    pts[tree.begin[c]:tree.end[c]], tree.box_lo[c],
                    tree.box_hi[c], p)
            h2.rank[c] = grid[c].shape[0]
        if lv > top:
            p_up = p0 + (tree.depth - lv + 1) // 2
            for c in tree.levels[lv]:
                par = tree.parent[c]
                h2.transfer[c] = interpolation_matrix(
                    grid[c], tree.box_lo[par], tree.box_hi[par], p_up)
    for lv in partition.levels():
        for s, t in partition.admissible_leaves[lv]:
            h2.coupling[(s, t)] = eval_kernel(spec, grid[s], grid[t])
    return h2


def _stacked_basis(h2, c):
    if h2.tree.is_leaf(c):
        return h2.leaf_basis[c]
    a, b = h2.tree.children(c)
    return np.vstack([h2.transfer[a], h2.transfer[b]])


def _store_basis(h2, c, q):
    if h2.tree.is_leaf(c):
        h2.leaf_basis[c] = q
        return
    a, b = h2.tree.children(c)
    ka = h2.rank[a]
    h2.transfer[a] = np.ascontiguousarray(q[:ka])
    h2.transfer[b] = np.ascontiguousarray(q[ka:])


def _qr_sweep(h2, index, top, depth):
    for lv in range(depth, top - 1, -1):
        for c in h2.tree.levels[lv]:
            q, r = np.linalg.qr(_stacked_basis(h2, c), mode="reduced")
            _store_basis(h2, c, q)
            h2.rank[c] = q.shape[1]
            for key, flip in index[lv].get(c, ()):
                h2.coupling[key] = (h2.coupling[key] @ r.T if flip
                                    else r @ h2.coupling[key])
            if c in h2.transfer:
                h2.transfer[c] = r @ h2.transfer[c]


def orthogonalize_recompress(h2, eps):
    part = h2.partition
    top = part.top_level
    if top is None:
        return h2
    depth = h2.tree.depth
    index = {lv: part.coupling_index(lv) for lv in part.levels()}
    _qr_sweep(h2, index, top, depth)
    weight_kept = {}
    for lv in range(top, depth + 1):
        for c in h2.tree.levels[lv]:
            blocks = [h2.coupling[key].T if flip else h2.coupling[key]
                      for key, flip in index[lv].get(c, ())]
            par = h2.tree.parent[c]
            if c in h2.transfer and weight_kept[par].size:
                blocks.append(h2.transfer[c] * weight_kept[par])
            if blocks:
                u, sig, _ = np.linalg.svd(np.hstack(blocks), full_matrices=False)
                cut = eps * sig[0] if sig.size else 0.0
                k = int(np.sum(sig > cut))
            else:
                u = np.zeros((h2.rank[c], 0))
                sig = np.zeros(0)
                k = 0
            uk = u[:, :k]
            _store_basis(h2, c, _stacked_basis(h2, c) @ uk)
            if c in h2.transfer:
                h2.transfer[c] = uk.T @ h2.transfer[c]
            for key, flip in index[lv].get(c, ()):
                h2.coupling[key] = (h2.coupling[key] @ uk if flip
                                    else uk.T @ h2.coupling[key])
            weight_kept[c] = sig[:k]
            h2.rank[c] = k
    _qr_sweep(h2, index, top, depth)
    return h2


# --------------------------------------------------------------------------
# symmetric low-rank update (h2core.py:333-392, kernels.py:89-96)
# --------------------------------------------------------------------------

def make_low_rank_factor(n, rank, seed):
    """n x rank Philox(seed) normals / sqrt(n) (kernels.py:89-96)."""
    return np.random.Generator(np.random.Philox(seed)).standard_normal((n, rank)) / np.sqrt(n)


def _range_basis(resid, scale):
    # orthonormal basis of resid's numerically significant range
    if resid.shape[1] == 0:
        return np.zeros((resid.shape[0], 0))
    u, sig, _ = np.linalg.svd(resid, full_matrices=False)
    return u[:, :int(np.sum(sig > 1e-12 * max(scale, 1e-300)))]


def absorb_low_rank(h2, w, eps):
    """A <- A + W W^T inside the H2 representation, in place, then
    recompression at eps.  Dense blocks take the explicit term; every
    cluster's basis is widened (bottom-up, in coefficient space above the
    leaves) until it reproduces its rows of W exactly, and the coupling
    blocks take the projected cross terms."""
    w = np.asarray(w, dtype=np.float64)
    if w.ndim != 2 or w.shape[0] != h2.n:
        raise ValueError("update factor must be n x r")
    tree, part = h2.tree, h2.partition
    for (s, t) in list(h2.dense):
        h2.dense[(s, t)] = h2.dense[(s, t)] + w[tree.begin[s]:tree.end[s]] @ w[tree.begin[t]:tree.end[t]].T
    if part.top_level is None:
        return h2
    coef = {}     # cluster -> its rows of W in its (widened) basis coordinates
    for lv in range(tree.depth, part.top_level - 1, -1):
        widened = {}
        for c in tree.levels[lv]:
            if tree.is_leaf(c):
                rows = w[tree.begin[c]:tree.end[c]]
            else:
                a, b = tree.children(c)
                rows = np.vstack([coef[a], coef[b]])
            basis = _stacked_basis(h2, c)
            inside = basis.T @ rows
            extra = _range_basis(rows - basis @ inside, float(np.linalg.norm(rows)))
            _store_basis(h2, c, np.hstack([basis, extra]))
            h2.rank[c] += extra.shape[1]
            widened[c] = extra.shape[1]
            coef[c] = np.vstack([inside, extra.T @ rows])
        for c in tree.levels[lv]:
            if widened[c] and c in h2.transfer:
                t = h2.transfer[c]
                h2.transfer[c] = np.vstack([t, np.zeros((widened[c], t.shape[1]))])
    for (s, t), blk in list(h2.coupling.items()):
        grown = np.zeros((h2.rank[s], h2.rank[t]))
        grown[:blk.shape[0], :blk.shape[1]] = blk
        h2.coupling[(s, t)] = grown + coef[s] @ coef[t].T
    return orthogonalize_recompress(h2, eps)


def h2_nbytes(h2):
    return sum(blk.nbytes for store in
               (h2.leaf_basis, h2.transfer, h2.coupling, h2.dense)
               for blk in store.values())


# --------------------------------------------------------------------------
# one-call problem construction (harness.py:86-194 restated)
# --------------------------------------------------------------------------

def build_problem(name, n, **overrides):
    """(tree, partition, spec, h2, params) for a named problem row.

    `overrides` may replace any row field (e.g. dim=2, kappa=0.0, eps=...).
    """
    if name not in PROBLEMS:
        raise ValueError(f"unknown problem {name!r}; choose from {sorted(PROBLEMS)}")
    prm = dict(PROBLEMS[name])
    prm.update({k: v for k, v in overrides.items() if v is not None})
    # LAPACK results depend on the BLAS thread count; one thread keeps the
    # operator bit-identical to the reference's
    with threadpool_limits(1):
        return _build(prm, n)


# wall seconds of the last build's stages (construction, compression and,
# for the low-rank row, the update) -- the harness reports them separately
LAST_BUILD_TIMINGS = {}


def _build(prm, n):
    import time
    t0 = time.perf_counter()
    points, counts = generate_uniform_grid(n, prm["dim"])
    h = 1.0 / max(counts)
    tree = build_cluster_tree(points, prm["m"])
    part = dual_tree_traversal(tree, prm["eta"])
    spec = KernelSpec(family=prm["family"], dim=prm["dim"],
                      corr_length=prm["corr_length"], kappa=prm["kappa"],
                      diag_value=default_diag_value(prm["family"], h),
                      alpha_r=prm["alpha_r"])
    h2 = build_h2(tree, part, spec, prm["p0"])
    t1 = time.perf_counter()
    h2 = orthogonalize_recompress(h2, prm["eps"])
    t2 = time.perf_counter()
    LAST_BUILD_TIMINGS.clear()
    LAST_BUILD_TIMINGS.update(construction=t1 - t0, compression=t2 - t1)
    if prm.get("lru_rank", 0) > 0:
        h2 = absorb_low_rank(h2, make_low_rank_factor(n, prm["lru_rank"], prm.get("seed", 7)), prm["eps"])
        LAST_BUILD_TIMINGS["low_rank_update"] = time.perf_counter() - t2
    return tree, part, spec, h2, prm


def rhs_for(h2, seed=7, nrhs=None):
    """The harness's synthetic right-hand side x_ref ~ Philox(seed) normal
    (harness.py:207-209); b is formed by the caller with matvec."""
    gen = np.random.Generator(np.random.Philox(seed))
    if nrhs is None:
        return gen.standard_normal(h2.n)
    return gen.standard_normal((h2.n, nrhs))
