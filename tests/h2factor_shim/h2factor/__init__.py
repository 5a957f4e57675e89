"""`h2factor` import alias over the B200 package: the
binding a maintainer would install to run the reference's own callers and
tests unchanged on the device path.  Only the public names of the path and
of the input construction are re-exported; nothing here computes."""
from paper_2509_11152_b200 import (FactorizationError, H2Factorization, estimate_norm2, factorize, matvec,  # noqa: F401
                                   refined_solve, solve, solve_multi)
