"""Seeded synthetic input streams shared by the oracle tests, the GPU tests and bench.py.

This package holds configuration records and random-number generation only.  It does
NOT implement any step of the STR/rSTR method (no unfoldings, subchains, Grams, solves
or updates): the generator builds data tensors from its own TR cores with plain numpy
matrix products, and both the oracle (``oracle/``) and the CUDA path
(``paper_2307_00719_b200``) consume its output as opaque arrays.
"""
from .configs import CONFIGS, StreamConfig, get_config  # noqa: F401
from .gen import Stream, make_stream  # noqa: F401
