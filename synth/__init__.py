"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the method (no attention, no merge, no copy
semantics, no allocation policy): it only draws random values, lays requests out in
paged pools the way a serving engine would have left them, and poisons unused memory.
Both ``oracle`` (tests) and ``paper_2510_13223_b200`` (tests/bench) consume its output.
"""
from .workload import *  # noqa: F401,F403
