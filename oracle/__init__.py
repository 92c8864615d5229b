"""Test infrastructure: the fp64 CPU oracle (see ns_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product path must never import it.
"""
from .ns_oracle import *  # noqa: F401,F403
