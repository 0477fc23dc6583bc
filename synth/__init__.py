"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no TTM, Gram, eigensolve, core
or fit).  It only draws the random inputs the paper's workloads are made of:

* COO nonzero positions and values (uniform-distinct, Bernoulli-per-cell, and
  bounded-Zipf skewed), and
* random orthonormal initial factors (the north star's "random orthonormal
  init factors from the seed").

See DESIGN.md "Input recipe" for the per-config parameters and the readings
(SURVEY.md §8(c) A11–A14) that fix the ambiguous parts.
"""
from .generators import (  # noqa: F401
    CONFIGS,
    bernoulli_dense,
    bernoulli_coo,
    bernoulli_coo_slabs,
    make_config,
    random_orthonormal,
    sp_random_init,
    uniform_distinct_coo,
    zipf_coo,
)
