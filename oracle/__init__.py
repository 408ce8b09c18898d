"""CPU oracle for Continuum's trace-replay hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product (paper_2511_02230_b200) never does.

Parity status: every function here is pinned by
`-m "not gpu"` tests against the paper's worked examples, closed forms, invariants
or brute force; the paper's end-to-end JCT gains are "parity
unpinned" (they need the paper's traces and GPUs) and are not computed here.
"""
from .oracle import *  # noqa: F401,F403
