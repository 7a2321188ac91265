"""CPU oracle of the reference's APSP arithmetic -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  It is the checker and the timed CPU baseline, never a product path.
"""
from .oracle import *  # noqa: F401,F403
