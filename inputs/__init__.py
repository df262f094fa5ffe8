"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the WASABI method (no PSFs, no wavelet, no
selection, no binning): only the configuration constants of BASELINE.json's
configs and the seeded random draws of object points.  See DESIGN.md §3 for the
recipe.
"""
from .generators import CONFIGS, Config, make_points, value_noise  # noqa: F401
