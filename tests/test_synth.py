"""The seeded input generators (synth/, shared by the oracle and the CUDA path).

The Zipf generator has a fast path (harmonic-asymptote inverse CDF + hash
dedup) and a torch-device path used for config 5; both must reproduce the
plain definition (searchsorted inverse CDF, first distinct cells in draw
order, reading A11/A12) exactly."""
import numpy as np

import synth.generators as G


def plain_zipf_coo(dims, nnz, rng, batch):
    """Reading A11/A12 written out: searchsorted inverse CDF per mode, np.unique
    with first occurrences, stop once nnz distinct cells exist."""
    def draw(I):
        w = 1.0 / np.arange(1, I + 1, dtype=np.float64)
        cdf = np.cumsum(w)
        cdf /= cdf[-1]
        return np.minimum(np.searchsorted(cdf, rng.random(batch), side="right"), I - 1)

    keys = np.empty(0, dtype=np.int64)
    while keys.size < nnz:
        k = None
        for I in dims:
            g = draw(I).astype(np.int64)
            k = g if k is None else k * I + g
        allk = np.concatenate([keys, k])
        _, first = np.unique(allk, return_index=True)
        keys = allk[np.sort(first)]
    keys = keys[:nnz]
    idx = G._decode(keys, dims)
    vals = np.log1p(rng.geometric(0.3, size=nnz).astype(np.float64)).astype(np.float32)
    return idx, vals


def test_zipf_paths_match_plain_definition():
    for dims, nnz, batch in (((50, 60, 7), 2000, 1 << 10), ((5000, 300, 40), 40_000, 1 << 14)):
        ref = plain_zipf_coo(dims, nnz, np.random.default_rng(5), batch)
        fast = G.zipf_coo(dims, nnz, np.random.default_rng(5), batch=batch)
        dev = G.zipf_coo(dims, nnz, np.random.default_rng(5), batch=batch, device="cpu")
        for got in (fast, dev):
            assert all(np.array_equal(a, b) for a, b in zip(got[0], ref[0]))
            assert np.array_equal(got[1], ref[1])
        # distinct cells, Zipf head at index 0, values log(1+c) >= log 2 (reading A13)
        keys = ref[0][0] * dims[1] * dims[2] + ref[0][1] * dims[2] + ref[0][2]
        assert np.unique(keys).size == nnz
        assert np.argmax(np.bincount(ref[0][0])) == 0
        assert ref[1].min() >= np.float32(np.log(2.0))


def test_bounded_zipf_inverse_cdf_exact():
    for I in (1, 2, 3, 17, 5000, 50000):
        u_rng, z_rng = np.random.default_rng(I), np.random.default_rng(I)
        w = 1.0 / np.arange(1, I + 1)
        cdf = np.cumsum(w)
        cdf /= cdf[-1]
        ref = np.minimum(np.searchsorted(cdf, u_rng.random(20000), side="right"), I - 1)
        assert np.array_equal(G._bounded_zipf(I, 20000, z_rng), ref)
