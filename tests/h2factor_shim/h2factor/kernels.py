from paper_2509_11152_b200.problem import KernelSpec, default_diag_value, make_low_rank_factor  # noqa: F401
