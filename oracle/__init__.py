"""CPU oracle for the HATA decode hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package.  See hata_oracle.py for the algorithm and its
citations into the paper.
"""
from .hata_oracle import *  # noqa: F401,F403
from . import hata_oracle  # noqa: F401
