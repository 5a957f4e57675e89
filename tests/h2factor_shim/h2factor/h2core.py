from paper_2509_11152_b200.h2core import estimate_norm2, matvec  # noqa: F401
from paper_2509_11152_b200.problem import H2Matrix, absorb_low_rank, build_h2, h2_nbytes, orthogonalize_recompress  # noqa: F401
