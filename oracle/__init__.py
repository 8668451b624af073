"""KVComm CPU oracle (float64 NumPy) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  It shares no code with paper_2510_12872_b200/.
"""
from .kvcomm_oracle import *  # noqa: F401,F403
