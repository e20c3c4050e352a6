"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

Holds no arithmetic of the method (see ``synth/workloads.py`` header)."""
from .workloads import *  # noqa: F401,F403
