from paper_2509_11152_b200.factorization import (FILL_DROP_FACTOR, PIVOT_RTOL, ClusterFactor,  # noqa: F401
                                                 FactorizationError, H2Factorization, LevelRecord, factorize)
