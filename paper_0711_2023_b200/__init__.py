"""B200-native HOOI / Multislice-Projection hot path (arxiv/paper_0711_2023).

The compute lives in ``libtucker.so`` (CUDA, sm_100a) behind the C-ABI in
``include/tucker.h``; :mod:`paper_0711_2023_b200.capi` is the ctypes binding.
"""
from .capi import (  # noqa: F401
    Tucker,
    TuckerError,
    core_and_fit,
    hooi_sweep,
    mp_sweep,
    tucker_debug_eig,
    tucker_debug_gram,
    tucker_debug_ttmc,
    tucker_free,
    tucker_init,
    tucker_set_factors,
    tucker_stats,
)
