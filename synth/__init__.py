"""Seeded synthetic input generators (no method arithmetic); see workloads.py."""
from .workloads import *  # noqa: F401,F403
