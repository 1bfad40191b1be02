"""CPU oracle for arXiv 1808.02937 -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.  It shares no code with
paper_1808_02937_b200/ (the product path); both read their inputs from
fde_inputs/, which holds no arithmetic of the method.
"""
from .oracle import *  # noqa: F401,F403
