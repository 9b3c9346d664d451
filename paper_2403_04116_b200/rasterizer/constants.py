"""Blend constants of the reference (kernels_py.py:13-19, frontend.py:32-36)."""

TILE_SIZE = 16
POWER_CUTOFF = -30.0
TRANSMITTANCE_FLOOR = 1e-4
SIGMA_CLAMP = 0.99
CUTOFF_SIGMA = 7.5
