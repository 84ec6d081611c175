"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This package holds NONE of the method's arithmetic (no rolling hash, no
matching, no RoPE, no scoring).  It only draws token ids, sensitivity masks,
span lists, KV payload values and attention matrices from fixed seeds, with
the shapes of the paper's workloads.
"""
from .gen import *  # noqa: F401,F403
