"""Seeded synthetic workloads shared by the oracle tests and the CUDA path.

This package holds ONLY input generation (observation positions, field values,
configuration records).  It contains none of the method's arithmetic (no GP
posterior, no bound, no Monte Carlo): per the build rules it is the one module
both `oracle/` and `paper_2512_12442_b200/` may consume.

The configurations mirror BASELINE.json configs c1..c5 (see DESIGN.md §3 for the
readings where BASELINE.json is silent) plus small ragged parity cases.
"""
from .configs import CONFIGS, Config, get_config  # noqa: F401
from .gen import generate, Workload  # noqa: F401
