"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds input generation only (matrices, orderings, initial block
partitions, right-hand sides) -- none of the BILU arithmetic.  Recipes: DESIGN.md
"Input recipe" (from SURVEY.md 8(d) and BASELINE.json configs).
"""
from .configs import CONFIGS, make_config, Problem  # noqa: F401
