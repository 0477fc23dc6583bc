"""Multi-GPU host logic on CPU.

The library shards HOOI by contiguous mode-n slice ranges and MP by ranges of
each term's slice index, and sums partial results with allreduces.  Here
(no GPU): the shard rule itself (tucker_shard_bounds, host-only C-ABI) and,
over a world_size-2 gloo process group, the exchange arithmetic -- each rank
computes only its shard with the fp64 oracle, the allreduces combine them, and
the result must equal the unsharded oracle.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tucker_oracle as O
from synth import random_orthonormal, uniform_distinct_coo


@pytest.fixture(scope="module")
def capi():
    from paper_0711_2023_b200 import capi as c
    return c


def test_shard_bounds_rule(capi):
    rng = np.random.default_rng(3)
    for n, world in ((0, 1), (0, 3), (1, 4), (7, 2), (100, 8), (1000, 3)):
        w = rng.exponential(size=n) * (rng.random(n) < 0.8)
        b = capi.shard_bounds(w, world)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
        if n:
            pre = np.concatenate([[0.0], np.cumsum(w)])
            T = pre[-1]
            for r in range(1, world):
                # within one item of the ideal split point
                assert abs(pre[b[r]] - r * T / world) <= w.max() + 1e-9
    assert list(capi.shard_bounds([1] * 8, 2)) == [0, 4, 8]
    assert list(capi.shard_bounds([0, 0, 3, 0, 0, 3, 0], 2)) == [0, 3, 7]
    with pytest.raises(capi.TuckerError):
        capi.shard_bounds([1.0, -1.0], 2)


def _rank_main(rank, world, port, dims, nnz, core, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_0711_2023_b200 import capi

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        dist.all_reduce(t)
        return t.numpy()

    idx, vals = uniform_distinct_coo(dims, nnz, np.random.default_rng(21))
    U0 = [random_orthonormal(I, J, np.random.default_rng(22 + k)) for k, (I, J) in enumerate(zip(dims, core))]
    T = O.SparseTensor(dims, idx, vals)
    U = [np.asarray(u, dtype=np.float64) for u in U0]
    N = len(dims)
    out = {}
    for n in range(N):
        # HOOI: this rank's slices of mode n (work = nnz per slice, the shard rule)
        b = capi.shard_bounds(np.bincount(idx[n], minlength=dims[n]).astype(float), world)
        sel = (idx[n] >= b[rank]) & (idx[n] < b[rank + 1])
        Tr = O.SparseTensor(dims, [i[sel] for i in idx], vals[sel])
        Yr = O.ttm_chain_unfold(Tr, U, n)  # rows outside the shard are zero
        P = Yr.shape[1]
        if P >= dims[n]:
            Y = allreduce(Yr)  # Y Y^T route: disjoint rows gathered by the sum
            Un, _ = O.leading_eigenvectors(Y @ Y.T, core[n])
        else:
            S = allreduce(Yr.T @ Yr)  # Y^T Y route: partial Grams summed
            w, V = np.linalg.eigh(S)
            o = np.argsort(-w)[: core[n]]
            Ur = Yr @ V[:, o] / np.sqrt(w[o])  # this rank's rows of U
            Un = np.linalg.qr(allreduce(Ur))[0]
        Yfull = O.ttm_chain_unfold(T, U, n)
        Uo, _ = O.leading_eigenvectors(Yfull @ Yfull.T, core[n])
        out["hooi%d" % n] = O.projector_distance(Un, Uo)
        # MP term (n, m): slices = the modes not in {n, m}; partial M_n summed
        M = np.zeros((dims[n], dims[n]))
        for m in range(N):
            if m == n:
                continue
            rest = [k for k in range(N) if k not in (n, m)]
            mk = np.zeros(nnz, dtype=np.int64)
            for k in rest:
                mk = mk * dims[k] + idx[k]
            ns = int(np.prod([dims[k] for k in rest]))
            bs = capi.shard_bounds(np.bincount(mk, minlength=ns).astype(float), world)
            s2 = (mk >= bs[rank]) & (mk < bs[rank + 1])
            Ts = O.SparseTensor(dims, [i[s2] for i in idx], vals[s2])
            Wr = O.mp_term_unfold(Ts, U[m], n, m)
            M += Wr @ Wr.T
        out["mp%d" % n] = float(np.linalg.norm(allreduce(M) - O.mp_gram(T, U, n)) / np.linalg.norm(O.mp_gram(T, U, n)))
        U[n] = Uo  # Gauss-Seidel with the reference factor
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


@pytest.mark.parametrize("dims,nnz,core", [((30, 40, 50), 3000, (4, 5, 6)), ((80, 6, 7), 2500, (3, 2, 2)),
                                           ((9, 10, 11, 12), 2000, (2, 3, 2, 3))])
def test_sharded_exchange_gloo_world2(dims, nnz, core):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000)
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, dims, nnz, core, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for k, v in out.items():
        assert v < 1e-9, (k, v)
