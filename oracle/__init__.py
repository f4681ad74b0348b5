"""CPU oracle package (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package.  The product package
``paper_2503_08415_b200`` never imports it and shares no code with it.
"""
from .oracle import *  # noqa: F401,F403
