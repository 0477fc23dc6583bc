"""Slice Projection on the GPU (NEXT 3 of SURVEY.md §8(f); sp_sweep / sp_run)
against the fp64 oracle (oracle.sp_sweep, pinned to the dense slice loops of
Figs. 5-6 in tests/test_oracle_pins.py) from the same random-uniform,
column-normalised initial factor, and the paper's printed SP fits
(Tables 2 and 6: 3.934 % and 3.908 %, Delta_G < 1e-4, Eq. 11)."""
import json
import os

import numpy as np
import pytest

from oracle import tucker_oracle as O
from synth import bernoulli_dense, random_orthonormal, sp_random_init, uniform_distinct_coo

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def capi():
    import __graft_entry__
    __graft_entry__.build()
    from paper_0711_2023_b200 import capi as c
    return c


@pytest.mark.parametrize("dims,nnz,core", [((100, 100, 100), 10_000, (10, 10, 10)),
                                           ((37, 300, 53), 9_000, (5, 16, 7)),
                                           ((20, 22, 18, 16), 12_000, (4, 5, 3, 6))])
def test_sp_sweeps_match_oracle(capi, dims, nnz, core):
    idx, vals = uniform_distinct_coo(dims, nnz, np.random.default_rng(81))
    U0 = [random_orthonormal(I, J, np.random.default_rng(82 + k)) for k, (I, J) in enumerate(zip(dims, core))]
    C0 = sp_random_init(dims[-1], core[-1], np.random.default_rng(83)).astype(np.float32)
    T = O.SparseTensor(dims, idx, vals)
    ref = O.run_sp(T, U0[:-1] + [C0], core, 3)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        t.set_factor(len(dims) - 1, C0, check=False)
        fits, gn, _ = t.sp_sweep(3)
        _, U, fit = t.core_and_fit()
    assert np.max(np.abs(fits - np.asarray(ref["fits"]))) < 1e-5
    assert np.max(np.abs(gn / np.asarray(ref["gnorms"]) - 1)) < 1e-5
    for n in range(len(dims)):
        assert O.projector_distance(U[n].astype(np.float64), ref["U"][n]) < 1e-4, n


def test_set_factor_checks(capi):
    dims, core = (30, 31, 32), (3, 3, 3)
    idx, vals = uniform_distinct_coo(dims, 2000, np.random.default_rng(84))
    U0 = [random_orthonormal(I, J, np.random.default_rng(85 + k)) for k, (I, J) in enumerate(zip(dims, core))]
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        bad = np.ones((32, 3), dtype=np.float32)
        with pytest.raises(capi.TuckerError):
            t.set_factor(2, bad, check=True)  # not orthonormal
        t.set_factor(2, bad / np.sqrt(32), check=False)  # SP-style init accepted
        bad[0, 0] = np.nan
        with pytest.raises(capi.TuckerError):
            t.set_factor(2, bad, check=False)


@pytest.mark.parametrize("key", ["table2_250cube_J25", "table6_100pow4_J20"])
def test_paper_sp_fit_on_gpu(capi, key):
    g = json.load(open(os.path.join(HERE, "golden", "paper_fits.json")))
    case, tol = g[key], g["tolerance_pp"]
    dims, core = tuple(case["dims"]), tuple(case["core"])
    X = bernoulli_dense(dims, case["density"], np.random.default_rng(1))
    nz = np.nonzero(X)
    idx = [np.asarray(i, dtype=np.int32) for i in nz]
    vals = X[nz].astype(np.float32)
    del X
    U0 = [random_orthonormal(I, J, np.random.default_rng(60 + k)) for k, (I, J) in enumerate(zip(dims, core))]
    C0 = sp_random_init(dims[-1], core[-1], np.random.default_rng(7)).astype(np.float32)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        t.set_factor(len(dims) - 1, C0, check=False)
        fits = t.sp_run(50, 1e-4)
    assert abs(100 * fits[-1] - case["sp"]) < tol, (fits[-1], len(fits))


def test_hosvd_and_sp_bitwise_deterministic(capi):
    """Same inputs -> bit-identical factors, core and fits: the
    sparse Gram's pair sort + reduce-by-key and SP's single-term Gram have no
    atomics."""
    dims, core = (60, 70, 80), (6, 7, 8)
    idx, vals = uniform_distinct_coo(dims, 20_000, np.random.default_rng(91))
    U0 = [random_orthonormal(I, J, np.random.default_rng(92 + k)) for k, (I, J) in enumerate(zip(dims, core))]
    C0 = sp_random_init(dims[-1], core[-1], np.random.default_rng(93)).astype(np.float32)
    outs = []
    for _ in range(2):
        with capi.Tucker(dims, core, idx, vals, U0) as t:
            t.hosvd()
            Gh, Uh, fh = t.core_and_fit()
            t.set_factor(len(dims) - 1, C0, check=False)
            fits, gn, _ = t.sp_sweep(2)
            Gs, Us, fs = t.core_and_fit()
        outs.append((Gh, Uh, fh, fits, gn, Gs, Us, fs))
    for x, y in zip(*outs):
        if isinstance(x, list):
            assert all(np.array_equal(u, v) for u, v in zip(x, y))
        else:
            assert np.array_equal(np.asarray(x), np.asarray(y))


@pytest.mark.parametrize("dims,nnz,core", [((100, 100, 100), 10_000, (10, 10, 10)),
                                           ((20, 22, 18, 16), 12_000, (4, 5, 3, 6))])
def test_kept_w_buffers_across_algorithms(capi, dims, nnz, core):
    """W_n buffers are kept per (mode, term set) and not re-zeroed (their zero
    blocks depend only on the tensor): interleaving MP and SP on one handle
    must give bit-identical results to fresh handles (set_factors resets the
    warm-start slots, so every run starts cold)."""
    idx, vals = uniform_distinct_coo(dims, nnz, np.random.default_rng(91))
    U0 = [random_orthonormal(I, J, np.random.default_rng(92 + k)) for k, (I, J) in enumerate(zip(dims, core))]
    C0 = sp_random_init(dims[-1], core[-1], np.random.default_rng(93)).astype(np.float32)

    def mp(t):
        t.set_factors(U0)
        fits = t.mp_sweep(2)
        G, U, fit = t.core_and_fit()
        return fits, G, U

    def sp(t):
        t.set_factors(U0)
        t.set_factor(len(dims) - 1, C0, check=False)
        fits, gn, _ = t.sp_sweep(2)
        G, U, fit = t.core_and_fit()
        return fits, G, U

    def same(a, b):
        fa, Ga, Ua = a
        fb, Gb, Ub = b
        assert np.array_equal(fa, fb)
        assert np.array_equal(Ga, Gb)
        assert all(np.array_equal(x, y) for x, y in zip(Ua, Ub))

    with capi.Tucker(dims, core, idx, vals, U0) as t:
        mp1 = mp(t)
        sp1 = sp(t)
        mp2 = mp(t)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        mp_fresh = mp(t)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        sp_fresh = sp(t)
    same(mp1, mp2)
    same(mp1, mp_fresh)
    same(sp1, sp_fresh)


def test_unconverged_solve_is_reported(capi):
    """The sweeps read every mode's solver info once, at the end of the sweep:
    a solve that cannot converge (one outer iteration, tol 1e-15) must still
    surface as TUCKER_E_CONVERGE (with finite results); default options as 0."""
    dims, core = (100, 100, 100), (10, 10, 10)
    idx, vals = uniform_distinct_coo(dims, 10_000, np.random.default_rng(95))
    U0 = [random_orthonormal(I, J, np.random.default_rng(96 + k)) for k, (I, J) in enumerate(zip(dims, core))]
    h = capi.tucker_init(dims, core, idx, vals, U0, eig_max_iter=1, eig_tol=1e-15)
    try:
        fits, _, rc = capi.hooi_sweep(h, 2, want_stage=True)
        assert rc == capi.E_CONVERGE and np.all(np.isfinite(fits))
        capi.tucker_set_factors(h, U0)
        fits, _, rc = capi.mp_sweep(h, 2, want_stage=True)
        assert rc == capi.E_CONVERGE and np.all(np.isfinite(fits))
    finally:
        capi.tucker_free(h)
    h = capi.tucker_init(dims, core, idx, vals, U0)
    try:
        _, _, rc = capi.hooi_sweep(h, 2, want_stage=True)
        assert rc == 0
        capi.tucker_set_factors(h, U0)
        _, _, rc = capi.mp_sweep(h, 2, want_stage=True)
        assert rc == 0
    finally:
        capi.tucker_free(h)
