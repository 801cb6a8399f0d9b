"""Seeded synthetic inputs shared by the oracle and the GPU path.

This package holds NO arithmetic of the Krylov methods: it only builds the
matrices and right-hand sides of BASELINE.json's five configs (and scaled
variants of the same recipes for parity tests), so that the oracle and the
CUDA path consume identical bytes.  Recipes: DESIGN.md §"Input recipe".
"""

from .generators import *  # noqa: F401,F403
