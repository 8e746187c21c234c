"""Seeded synthetic-input generators shared by the oracle side and the CUDA
side (they hold none of the method's arithmetic; see gen/rng.py)."""
from . import configs, ct, rng  # noqa: F401
from .configs import CONFIGS, Config, spectrum  # noqa: F401
