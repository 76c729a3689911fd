"""CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  The product path
(paper_1805_12096_b200/) must never import it; tests/test_boundary.py checks
that.  See oracle/mnmt_oracle.c for the algorithm and its citations.
"""
from .oracle import *  # noqa: F401,F403
