"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and
bench.py.  Holds NONE of the method's arithmetic (no PRF, no tree, no
contraction): only random tables, target indices, payload multipliers beta and
the 32-byte DRBG seeds that Gen consumes (the random numbers the method draws
are passed in as inputs).  Recipe: DESIGN.md "Synthetic inputs".
"""
from .inputs import *  # noqa: F401,F403
