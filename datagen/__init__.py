"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the method (no kernel, no HSS, no ADMM):
only the config table and the PCG64 draws that produce (F_train, y_train,
F_test, y_test). Both `oracle/` and `paper_2108_04167_b200/` consume it; neither
is imported from here.
"""
from .configs import CONFIGS, get_config, beta_schedule  # noqa: F401
from .synth import generate  # noqa: F401
