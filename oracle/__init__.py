"""CPU double-precision oracle for GPU-FV Fisher-vector encoding (arXiv 1604.03498).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs.  The product package (paper_1604_03498_b200) never
imports it, and it never imports the product package.  See oracle/fv_oracle.c for the arithmetic and
the PAPER.md passages each function follows.

Parity status: every function here is pinned by tests/test_oracle.py (closed forms, invariants,
mpmath brute force, scipy / numpy library routines); none is "parity unpinned".  The §8(f) rows are
plain numpy in oracle/oracle.py: ``score`` (NEXT-4, linear decision values), ``loglik_rows`` /
``em_step`` (NEXT-3, diagonal-GMM EM with SPEC's floors), ``embed`` (NEXT-2, PCA + normalised xy).
"""
from .oracle import (  # noqa: F401
    NORM_IMPROVED,
    NORM_NONE,
    NORM_POWER_L2,
    accumulate,
    build,
    embed,
    em_step,
    em_step_blocked,
    encode,
    encode_batched,
    fv_from_stats,
    loglik_rows,
    max_threads,
    normalize,
    posteriors,
    score,
    stats,
    stats_batched,
    stats_blocked,
)
