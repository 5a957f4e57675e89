"""B200-native factorize/solve path of the strong-recursive-skeletonization
H2 direct solver (arXiv 2509.11152), a drop-in for the reference package's
path API (/root/reference/pkg/src/h2factor/__init__.py:11-26):

    factorize(h2, eps_lu, threads=1, norm_estimate=None) -> H2Factorization
    solve(fac, b) / solve_multi(fac, B) / refined_solve(h2, fac, b, steps=1)
    matvec(h2, x), estimate_norm2(h2, iters=30, seed=20240901)
    FactorizationError

Everything numeric runs in libh2f.so (C++ scheduler + sm_100a CUDA kernels).
`problem` holds the host-side input builder (tree, partition, H2 operator).
"""
from .factorization import (
    FILL_DROP_FACTOR,
    PIVOT_RTOL,
    ClusterFactor,
    FactorizationError,
    H2Factorization,
    LevelRecord,
    factorize,
)
from .h2core import estimate_norm2, matvec
from .problem import (
    PROBLEMS,
    BlockPartition,
    ClusterTree,
    H2Matrix,
    KernelSpec,
    build_cluster_tree,
    build_h2,
    build_problem,
    dual_tree_traversal,
    generate_uniform_grid,
    h2_nbytes,
    orthogonalize_recompress,
)
from .serialize import load_factorization, save_factorization
from .solve import refined_solve, refined_solve_multi, solve, solve_multi
from .structure import color_groups, greedy_coloring, level_graph, sparsity_constant

__version__ = "0.1.0"

__all__ = [
    "BlockPartition", "ClusterFactor", "ClusterTree", "FILL_DROP_FACTOR", "FactorizationError",
    "H2Factorization", "H2Matrix", "KernelSpec", "LevelRecord", "PIVOT_RTOL", "PROBLEMS",
    "build_cluster_tree", "build_h2", "build_problem", "color_groups", "dual_tree_traversal",
    "estimate_norm2", "factorize", "generate_uniform_grid", "greedy_coloring", "h2_nbytes",
    "level_graph", "load_factorization", "matvec", "orthogonalize_recompress", "save_factorization", "refined_solve", "refined_solve_multi", "solve", "solve_multi",
    "sparsity_constant", "__version__",
]
