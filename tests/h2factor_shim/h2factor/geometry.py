from paper_2509_11152_b200.problem import ClusterTree, build_cluster_tree, generate_uniform_grid  # noqa: F401
