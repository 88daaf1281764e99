"""Seeded synthetic workloads shared by the oracle tests, the GPU tests and bench.py.

This package holds ONLY input recipes: mesh sizes, coefficients and seeded random /
closed-form fields sampled at node coordinates.  It contains none of the method's
arithmetic (no operator, no quadrature, no solver), so that the CPU oracle
(``oracle/``) and the CUDA path (``paper_2112_04167_b200``) can both consume
identical arrays without sharing code.
"""
from .inputs import (  # noqa: F401
    CONFIGS,
    Config,
    config,
    gll_points_for_sampling,
    node_coords,
    rng,
    uniform_field,
)
