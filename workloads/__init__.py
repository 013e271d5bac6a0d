"""Seeded synthetic input generators shared by the oracle tests, the GPU tests
and bench.py.

This module holds NO arithmetic of the ACI method (no prrLU, frames, Π
assembly or cross interpolation). It only builds the input tensor trains of
BASELINE.json configs[0..4], the random initial guess y_init,
and the random sample multi-indices used for error estimates.
Recipes and readings are in DESIGN.md §3.
"""
from .generators import (  # noqa: F401
    TT, cosine_sum_tt, plane_wave_tt, random_tt, gaussian3d_tt, random_init,
    sample_indices, make_config, CONFIG_NAMES,
)
