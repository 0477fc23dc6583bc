"""HOOI at tensor orders 2 and 5..8 (HOOI takes orders 2-8; Fig. 4 P:606-644 is
written for any N, order 2 is the matrix case P:371-374).  The GPU path for these orders is
gen.cu (sorted COO per mode, one CTA per slice); orders 3 and 4 keep the CSF kernels.  Same
bars as tests/test_gpu_parity.py: Y_(n) <= 1e-4 relative Frobenius, factors <= 1e-4
projector distance, fits <= 1e-5, core <= 1e-4 after Procrustes alignment.  MP / SP are
defined for orders 3 and 4 only (reading A18): E_ARG."""
import numpy as np
import pytest

from oracle import tucker_oracle as O
from synth import random_orthonormal, uniform_distinct_coo

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi():
    import __graft_entry__
    __graft_entry__.build()
    from paper_0711_2023_b200 import capi as c
    return c


def case(dims, nnz, core, seed=11):
    rng = np.random.default_rng(seed)
    idx, vals = uniform_distinct_coo(dims, nnz, rng)
    frng = np.random.default_rng(seed + 1)
    U0 = [random_orthonormal(I, J, frng) for I, J in zip(dims, core)]
    return idx, vals, U0


def align_core(G, U, Uo):
    Ga = np.asarray(G, dtype=np.float64)
    for n in range(len(U)):
        a, _, bt = np.linalg.svd(np.asarray(U[n], dtype=np.float64).T @ Uo[n])
        Ga = O.ttm(Ga, (a @ bt).T, n)
    return Ga


SHAPES = [
    ((300, 200), 6_000, (6, 6)),                          # order 2 (J_1 = J_2 is forced: J_n <= prod_{q != n} J_q)
    ((60, 45), 900, (5, 5)),                              # order 2, ragged; both modes take the Y^T Y route
    ((40, 10, 9, 11, 8), 6_000, (3, 2, 3, 2, 2)),         # order 5: mode 1 takes Y^T Y (P = 24 < 40)
    ((9, 8, 7, 8, 6, 7), 8_000, (2, 3, 2, 2, 2, 3)),      # order 6
    ((5, 4, 5, 4, 5, 4, 5, 4), 10_000, (2, 2, 2, 2, 2, 2, 2, 2)),  # order 8 (P = 128 columns)
]


@pytest.mark.parametrize("dims,nnz,core", SHAPES)
def test_generic_order_hooi(capi, dims, nnz, core):
    idx, vals, U0 = case(dims, nnz, core)
    T = O.SparseTensor(dims, idx, vals)
    N = len(dims)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        # Y_(n) of the first mode from U0 (Eq. 1 chained, Kolda column order)
        for n in (0, N - 1):
            Y = t.debug_ttmc(n)
            Yo = O.ttm_chain_unfold(T, U0, n)
            assert O.rel_frobenius(Y, Yo) < 1e-4, n
        t.set_factors(U0)
        fits = t.hooi_sweep(3)
        G, U, fit = t.core_and_fit()
    ref = O.run_hooi(T, U0, core, 3)
    for n in range(N):
        assert O.projector_distance(U[n], ref["U"][n]) < 1e-4, n
        assert np.abs(U[n].astype(np.float64).T @ U[n] - np.eye(core[n])).max() < 1e-5
    np.testing.assert_allclose(fits, ref["fits"], atol=1e-5)
    assert abs(fit - ref["fit"]) < 1e-5
    assert O.rel_frobenius(align_core(G, U, ref["U"]), ref["G"]) < 1e-4


def test_generic_order_rules(capi):
    dims, core = (12, 10, 9, 11, 8), (3, 2, 3, 2, 2)
    idx, vals, U0 = case(dims, 3_000, core)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        with pytest.raises(capi.TuckerError) as e:
            t.mp_sweep(1)
        assert e.value.code == 1  # E_ARG: MP is defined for orders 3 and 4
        with pytest.raises(capi.TuckerError) as e:
            t.sp_sweep(1)
        assert e.value.code == 1
    # duplicates / out of range / non-finite, as for orders 3-4
    idx_d = [np.concatenate([a, a[:1]]) for a in idx]
    with pytest.raises(capi.TuckerError) as e:
        capi.Tucker(dims, core, idx_d, np.concatenate([vals, vals[:1]]), U0)
    assert e.value.code == 3
    idx_o = [a.copy() for a in idx]
    idx_o[4][7] = dims[4]
    with pytest.raises(capi.TuckerError) as e:
        capi.Tucker(dims, core, idx_o, vals, U0)
    assert e.value.code == 2
    v = vals.copy()
    v[5] = np.inf
    with pytest.raises(capi.TuckerError) as e:
        capi.Tucker(dims, core, idx, v, U0)
    assert e.value.code == 4
    # explicit zeros are dropped: same result as without them
    v = vals.copy()
    v[::5] = 0
    keep = v != 0
    with capi.Tucker(dims, core, idx, v, U0) as t1, \
            capi.Tucker(dims, core, [a[keep] for a in idx], v[keep], U0) as t2:
        f1 = t1.hooi_sweep(2)
        f2 = t2.hooi_sweep(2)
        _, U1, _ = t1.core_and_fit()
        _, U2, _ = t2.core_and_fit()
    np.testing.assert_array_equal(f1, f2)
    for a, b in zip(U1, U2):
        np.testing.assert_array_equal(a, b)


def test_generic_order_deterministic(capi):
    dims, core = (9, 8, 7, 8, 6, 7), (2, 3, 2, 2, 2, 3)
    idx, vals, U0 = case(dims, 5_000, core, seed=3)
    outs = []
    for _ in range(2):
        with capi.Tucker(dims, core, idx, vals, U0) as t:
            f = t.hooi_sweep(2)
            G, U, fit = t.core_and_fit()
            outs.append((f, G, U))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    for a, b in zip(outs[0][2], outs[1][2]):
        np.testing.assert_array_equal(a, b)
