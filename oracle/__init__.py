"""TEST INFRASTRUCTURE — the plain, slow, fp64 CPU oracle for arXiv 2311.13147.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import,
call or execute anything under oracle/. The product package (paper_2311_13147_b200/) never does, and
the oracle never imports the product package: the two share no code, headers, helpers or constants.

Every function cites the PAPER.md passage (P:line) it follows. Pins (tests/test_oracle_*.py) tie the
oracle to values and identities the paper and mathematics fix. Parity status per function is listed in
DESIGN.md §3; no function here is "parity unpinned" except the Table 1/2 absolute values (not used).
"""
from .core import *        # noqa: F401,F403
from .lot import *         # noqa: F401,F403
from .sinkhorn import *    # noqa: F401,F403
from .srot import *        # noqa: F401,F403
from .twostage import *    # noqa: F401,F403
