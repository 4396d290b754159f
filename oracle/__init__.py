"""CPU oracle of the multistep BSDE scheme (arXiv 1909.13560).

TEST INFRASTRUCTURE ONLY: tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_1909_13560_b200``) never imports it and shares no code
with it.  See ``oracle/bsde_oracle.h`` for the passages each routine follows.
"""
from .oracle import (  # noqa: F401
    OracleError, build_oracle, gauss_hermite, gamma_row, balance_npts,
    spline_moments, spline_eval, thomas, Oracle, terminal, exact, driver, fd_weights, fd_deriv,
)
