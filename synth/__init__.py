"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no quantisation, no scoring, no
selection, no FFN): only shapes (``configs``) and seeded random draws
(``gen``).  It is the one piece of code both sides of a parity test may use
(DESIGN.md "Input recipe").
"""
from .configs import CONFIGS, ModelConfig, get_config  # noqa: F401
from .gen import (  # noqa: F401
    layer_weights,
    token_stream,
    layer_input_stream,
    sigma_down,
    seed_for,
)
