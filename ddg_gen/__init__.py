"""Seeded synthetic inputs (no method arithmetic) shared by oracle tests and the CUDA path."""
from .problems import Problem, make, CONFIGS, CONFIG_TEXT  # noqa: F401
