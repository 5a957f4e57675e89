from paper_2509_11152_b200.problem import BlockPartition, dual_tree_traversal, sparsity_constant  # noqa: F401
from paper_2509_11152_b200.structure import color_groups, greedy_coloring, level_graph  # noqa: F401
