"""Seeded generators for the BASELINE.json configs (no method arithmetic here).

Conventions:
* indices are 0-based int32, one array per mode, nonzeros in random (unsorted)
  order -- the library sorts them itself (PAPER.md P:854-861 sorts the COO file);
* values are fp32;
* factors are fp32 row-major I_n x J_n with orthonormal columns.
"""
from __future__ import annotations

import numpy as np

# BASELINE.json "configs", 1-based as in the survey.  seeds: tensor / factors
# (SURVEY.md §8(d) table "Seeds (proposed)").
CONFIGS = {
    1: dict(dims=(100, 100, 100), nnz=10_000, core=(10, 10, 10), sweeps=3,
            kind="uniform", seed=1, fseed=101),
    2: dict(dims=(1000, 1000, 1000), nnz=1_000_000, core=(50, 50, 50), sweeps=5,
            kind="uniform", seed=2, fseed=102),
    3: dict(dims=(2000, 2000, 2000), nnz=8_000_000, core=(100, 25, 10), sweeps=5,
            kind="uniform", seed=3, fseed=103),
    4: dict(dims=(200, 200, 200, 200), nnz=16_000_000, core=(20, 20, 20, 20),
            sweeps=5, kind="uniform", seed=4, fseed=104),
    5: dict(dims=(50_000, 50_000, 5_000), nnz=200_000_000, core=(100, 100, 50),
            sweeps=5, kind="zipf", seed=5, fseed=105),
}


def _decode(keys: np.ndarray, dims) -> list[np.ndarray]:
    """Row-major decode of linear cell keys into per-mode int32 indices."""
    out = []
    rem = keys.astype(np.int64, copy=True)
    for I in reversed(dims[1:]):
        out.append((rem % I).astype(np.int32))
        rem //= I
    out.append(rem.astype(np.int32))
    return out[::-1]


def uniform_distinct_coo(dims, nnz, rng: np.random.Generator):
    """`nnz` distinct cells drawn uniformly from prod(dims), values in (0,1].

    Reading A14: values are ``1 - U[0,1)`` so no explicit zero is produced.
    Positions: over-draw, unique, top up, then a uniformly random subset of
    exactly `nnz` keys, returned in random order.
    """
    total = int(np.prod(np.asarray(dims, dtype=np.float64)))
    if nnz > total:
        raise ValueError("nnz exceeds the number of cells")
    keys = np.empty(0, dtype=np.int64)
    draw = int(nnz * 1.05) + 16
    while keys.size < nnz:
        new = rng.integers(0, total, size=draw, dtype=np.int64)
        keys = np.unique(np.concatenate([keys, new]))
        draw = max(16, int((nnz - keys.size) * 1.2) + 16)
    pick = rng.choice(keys.size, size=nnz, replace=False)
    keys = keys[pick]  # random order
    idx = _decode(keys, dims)
    vals = (np.float32(1.0) - rng.random(nnz, dtype=np.float32)).astype(np.float32)
    return idx, vals


def bernoulli_dense(dims, density, rng: np.random.Generator) -> np.ndarray:
    """The paper's generator: every cell is nonzero
    with probability `density`, value uniform in (0,1].  Dense fp64 output."""
    mask = rng.random(dims) < density
    vals = 1.0 - rng.random(dims)
    return np.where(mask, vals, 0.0)


def bernoulli_coo_slabs(dims, density, seed: int, slab_cells: int = 1 << 25):
    """The paper's generator (every cell nonzero with probability `density`, value
    uniform in (0,1]) for tensors too large for a dense array (Table 2's
    750^3 and 1000^3: 4e8 / 1e9 cells): slabs of whole mode-1 indices, each drawn from
    its own stream seeded by (seed, slab).  Returns int32 COO + fp32 values."""
    dims = tuple(int(d) for d in dims)
    inner = int(np.prod(dims[1:]))
    per = max(1, slab_cells // inner)
    idx_parts, val_parts = [[] for _ in dims], []
    for s0 in range(0, dims[0], per):
        s1 = min(dims[0], s0 + per)
        r = np.random.default_rng([seed, s0])
        n = (s1 - s0) * inner
        mask = r.random(n) < density
        vals = (1.0 - r.random(n))[mask]
        lin = np.flatnonzero(mask)
        sub = np.unravel_index(lin, (s1 - s0,) + dims[1:])
        idx_parts[0].append((sub[0] + s0).astype(np.int32))
        for k in range(1, len(dims)):
            idx_parts[k].append(sub[k].astype(np.int32))
        val_parts.append(vals.astype(np.float32))
    return [np.concatenate(p) for p in idx_parts], np.concatenate(val_parts)


def bernoulli_coo(dims, density, rng: np.random.Generator):
    X = bernoulli_dense(dims, density, rng)
    nz = np.nonzero(X)
    idx = [a.astype(np.int32) for a in nz]
    return idx, X[nz].astype(np.float32)


def _bounded_zipf(I: int, size: int, rng, s: float = 1.0) -> np.ndarray:
    """Reading A11: P(k) ∝ 1/k^s on k=1..I, rank k -> index k-1.

    Inverse CDF: the index is searchsorted(cdf, u, side="right").  For s = 1
    the search starts from the harmonic-number asymptote H_k ≈ ln k + γ and is
    then corrected against the same cdf table, so the result is identical to
    the plain search (only faster: ~1e9 draws at config 5).
    """
    w = 1.0 / np.arange(1, I + 1, dtype=np.float64) ** s
    cdf = np.cumsum(w)
    H = cdf[-1]
    cdf /= H
    u = rng.random(size)
    if s != 1.0:
        return np.minimum(np.searchsorted(cdf, u, side="right"), I - 1).astype(np.int64)
    g = np.exp(u * H - 0.5772156649015329)
    g = np.clip(g.astype(np.int64) - 1, 0, I - 1)
    # exact fix-up: want cdf[g-1] <= u < cdf[g] (g = I-1 if u >= cdf[I-2])
    sel = np.nonzero((cdf[g] <= u) | ((g > 0) & (cdf[np.maximum(g - 1, 0)] > u)))[0]
    while sel.size:
        gs, us = g[sel], u[sel]
        up = (cdf[gs] <= us) & (gs < I - 1)
        dn = (gs > 0) & (cdf[np.maximum(gs - 1, 0)] > us)
        gs = gs + up - dn
        g[sel] = gs
        keep = (up | dn)
        sel = sel[keep]
    return g


def _zipf_coo_torch(dims, nnz, rng, batch, device):
    """zipf_coo on a torch device: the same numpy uniforms (same stream
    order), searchsorted against the same cdf tables and first-occurrence
    dedup by sort -- identical output, minutes -> seconds at config 5."""
    import torch

    cdfs = []
    for I in dims:
        w = 1.0 / np.arange(1, I + 1, dtype=np.float64)
        c = np.cumsum(w)
        c /= c[-1]
        cdfs.append(torch.from_numpy(c).to(device))
    keys = torch.empty(0, dtype=torch.int64, device=device)
    while keys.numel() < nnz:
        k = None
        for I, cdf in zip(dims, cdfs):
            u = torch.from_numpy(rng.random(batch)).to(device)
            g = torch.clamp(torch.searchsorted(cdf, u, right=True), max=I - 1)
            k = g if k is None else k * I + g
        allk = torch.cat([keys, k])
        uniq, inv = torch.unique(allk, sorted=True, return_inverse=True)
        first = torch.full((uniq.numel(),), allk.numel(), dtype=torch.int64, device=device)
        first.scatter_reduce_(0, inv, torch.arange(allk.numel(), device=device), "amin")
        keys = allk[torch.sort(first).values]
        del allk, uniq, inv, first, k
    keys = keys[:nnz].cpu().numpy()
    torch.cuda.empty_cache()
    idx = _decode(keys, dims)
    c = rng.geometric(0.3, size=nnz)
    vals = np.log1p(c.astype(np.float64)).astype(np.float32)
    return idx, vals


def zipf_coo(dims, nnz, rng: np.random.Generator, batch: int = 1 << 26, device=None):
    """Config 5: each mode index Zipf(1) independently, deduplicated.

    Reading A12: draw in batches until at least `nnz` distinct cells exist and
    keep the first `nnz` distinct cells in draw order.  Reading A13: values are
    log(1+c), c ~ Geometric(p=0.3) on {1,2,...}.  The dedup is hash based
    (pandas.unique keeps first occurrences in order).
    """
    total_bits = sum(int(np.ceil(np.log2(I))) for I in dims)
    assert total_bits <= 62
    if device is not None:
        return _zipf_coo_torch(dims, nnz, rng, batch, device)
    import pandas as pd

    parts = []
    n = 0
    seen = None
    while n < nnz:
        cols = [_bounded_zipf(I, batch, rng) for I in dims]
        k = cols[0]
        for I, c in zip(dims[1:], cols[1:]):
            k = k * I + c
        del cols
        u = pd.unique(k)
        del k
        if seen is not None:
            u = u[~pd.Series(u).isin(seen).to_numpy()]
        parts.append(u)
        n += u.size
        if n < nnz:
            seen = np.concatenate(parts) if len(parts) > 1 else parts[0]
    keys = np.concatenate(parts)[:nnz]
    del parts, seen
    idx = _decode(keys, dims)
    c = rng.geometric(0.3, size=nnz)
    vals = np.log1p(c.astype(np.float64)).astype(np.float32)
    return idx, vals


def random_orthonormal(I: int, J: int, rng: np.random.Generator) -> np.ndarray:
    """Q of a seeded Gaussian's QR with sign(diag R) folded in, as fp32
    (SURVEY.md §8(d) "U0 recipe"; north star "random orthonormal init")."""
    Q, R = np.linalg.qr(rng.standard_normal((I, J)))
    Q = Q * np.sign(np.diag(R))[None, :]
    return np.ascontiguousarray(Q.astype(np.float32))


def sp_random_init(I: int, J: int, rng: np.random.Generator) -> np.ndarray:
    """Slice Projection's initial last factor: uniform [0, 1]
    entries, columns normalised to unit length (not orthonormalised).  An input
    draw shared by the oracle and the CUDA path (fp64; cast for the GPU)."""
    C = rng.random((I, J))
    return C / np.linalg.norm(C, axis=0, keepdims=True)


def make_config(k: int, *, nnz: int | None = None, dims=None, core=None, device=None):
    """Materialise BASELINE.json config `k` (optionally resized for tests).

    `device` (e.g. "cuda") only accelerates the Zipf generator (config 5);
    the arrays returned are identical either way."""
    c = dict(CONFIGS[k])
    if dims is not None:
        c["dims"] = tuple(dims)
    if core is not None:
        c["core"] = tuple(core)
    if nnz is not None:
        c["nnz"] = int(nnz)
    rng = np.random.default_rng(c["seed"])
    if c["kind"] == "uniform":
        idx, vals = uniform_distinct_coo(c["dims"], c["nnz"], rng)
    else:
        idx, vals = zipf_coo(c["dims"], c["nnz"], rng, device=device)
    frng = np.random.default_rng(c["fseed"])
    U0 = [random_orthonormal(I, J, frng) for I, J in zip(c["dims"], c["core"])]
    c.update(idx=idx, vals=vals, U0=U0)
    return c
