"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This package holds NO arithmetic of the method (no control volumes, no
operators, no eigen-bases, no solves): it only produces the grid steps,
layer coefficients, block partitions, shift and right-hand sides that
BASELINE.json's configs describe, following SURVEY.md §8(d)'s recipe.
Both the oracle (``oracle/``) and the CUDA path (``paper_1909_01299_b200``)
consume its output; neither is imported here.
"""
from .configs import Problem, make_problem, CONFIG_NAMES, shrunken, anomaly  # noqa: F401
