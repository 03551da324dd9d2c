"""Periodic FMM on the B200: drop-in for lambdafmm.fmm (reference fmm/__init__.py:3-4)."""

from .solver import PeriodicSolver, SolveResult, SolverConfig  # noqa: F401
