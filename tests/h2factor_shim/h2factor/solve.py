from paper_2509_11152_b200.solve import refined_solve, solve, solve_multi  # noqa: F401
