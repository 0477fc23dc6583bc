"""The sharded (multi-GPU) code path on one GPU: a handle created with an
NCCL id and world == 1 runs every exchange step of the sharded sweep (row /
slice shards, Y / S / U / G / M_n allreduces over a 1-rank NCCL communicator)
and must reproduce the unsharded handle exactly (a 1-rank allreduce is a copy
and the shards are the full ranges).  The world > 1 arithmetic is covered on
CPU by tests/test_multigpu_cpu.py (gloo, world 2)."""
import numpy as np
import pytest

from synth import random_orthonormal, uniform_distinct_coo

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi():
    import __graft_entry__
    __graft_entry__.build()
    from paper_0711_2023_b200 import capi as c
    return c


@pytest.mark.parametrize("dims,nnz,core", [
    ((100, 100, 100), 10_000, (10, 10, 10)),   # Y Y^T route
    ((37, 300, 53), 9_000, (5, 16, 7)),        # Y^T Y route on modes 1, 3
    ((20, 22, 18, 16), 12_000, (4, 5, 3, 6)),  # order 4
])
def test_sharded_path_world1_matches_unsharded(capi, dims, nnz, core):
    rng = np.random.default_rng(31)
    idx, vals = uniform_distinct_coo(dims, nnz, rng)
    U0 = [random_orthonormal(I, J, np.random.default_rng(40 + k)) for k, (I, J) in enumerate(zip(dims, core))]
    nid = capi.nccl_unique_id()
    assert len(nid) == 128
    res = []
    for kw in ({}, {"rank": 0, "world": 1, "nccl_id": nid}):
        with capi.Tucker(dims, core, idx, vals, U0, **kw) as t:
            hooi, mpi = t.shard_info()
            assert all(lo == 0 and hi > 0 for lo, hi in hooi)
            fh = t.hooi_sweep(2)
            Gh, Uh, fith = t.core_and_fit()
            t.set_factors(U0)
            fm = t.mp_sweep(2)
            Gm, Um, fitm = t.core_and_fit()
            res.append((fh, Gh, Uh, fith, fm, Gm, Um, fitm))
    a, b = res
    for x, y in zip(a, b):
        if isinstance(x, list):
            for u, v in zip(x, y):
                assert np.array_equal(u, v)
        else:
            assert np.array_equal(np.asarray(x), np.asarray(y))
