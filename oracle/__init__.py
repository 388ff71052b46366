"""TEST INFRASTRUCTURE ONLY - the CPU oracle of the NineToothed kernel set.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package, and only as the checker (or the
reported CPU baseline), never as the thing measured or shipped.  The product
path (paper_2507_11978_b200) must never import it.
"""
from .ntb_oracle import *  # noqa: F401,F403
