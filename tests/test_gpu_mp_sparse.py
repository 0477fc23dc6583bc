"""MP's multislice Gram without the dense W (mp_sparse.cu) and the host-driven
eigensolver for large d (eig_large.cu), forced on small inputs so that the fp64
oracle checks them element by element (the library picks them on its own only when
W_n would not fit, i.e. BASELINE config 5; tests/test_gpu_config5.py covers that).

  M_n                 <= 1e-5 relative Frobenius (3xTF32 products, fp64 accumulation)
  factors             <= 1e-4 projector distance after full MP / SP sweeps
  fits                <= 1e-5 absolute
  eigenvectors        <= 1e-5 projector distance vs LAPACK (eig_large)
"""
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


def case(dims, nnz, core, seed=17, fseed=18):
    rng = np.random.default_rng(seed)
    idx, vals = uniform_distinct_coo(dims, nnz, rng)
    frng = np.random.default_rng(fseed)
    U0 = [random_orthonormal(I, J, frng) for I, J in zip(dims, core)]
    return idx, vals, U0


SHAPES = [
    ((100, 100, 100), 10_000, (10, 10, 10)),     # config 1
    ((100, 110, 120), 13_200, (10, 11, 12)),     # non-cubic (Appendix `test`)
    ((37, 300, 53), 9_000, (5, 16, 7)),          # ragged; slices of up to 300 rows (3 tiles)
    ((300, 280, 12), 30_000, (9, 7, 5)),         # few slices with many rows each (multi-tile products)
]


@pytest.mark.parametrize("dims,nnz,core", SHAPES)
def test_sparse_mp_gram_parity(capi, monkeypatch, dims, nnz, core):
    monkeypatch.setenv("TUCKER_MP_SPARSE", "1")
    idx, vals, U0 = case(dims, nnz, core)
    T = O.SparseTensor(dims, idx, vals)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        for n in range(3):
            M = t.debug_gram(1, n)
            Mo = O.mp_gram(T, U0, n)
            assert O.rel_frobenius(M, Mo) < 1e-5, n
            rows = [0, dims[n] // 2, dims[n] - 1]
            np.testing.assert_allclose(t.debug_gram_rows(1, n, rows), Mo[rows], rtol=1e-5, atol=1e-5 * np.abs(Mo).max())


@pytest.mark.parametrize("dims,nnz,core", SHAPES)
@pytest.mark.parametrize("large_eig", [False, True])
def test_sparse_mp_sweeps_parity(capi, monkeypatch, dims, nnz, core, large_eig):
    """Full MP sweeps (and Slice Projection, the single-term variant) through the sparse
    Gram, optionally with the host-driven eigensolver, against the oracle."""
    monkeypatch.setenv("TUCKER_MP_SPARSE", "1")
    if large_eig:
        monkeypatch.setenv("TUCKER_EIG_LARGE", "1")
    idx, vals, U0 = case(dims, nnz, core)
    T = O.SparseTensor(dims, idx, vals)
    ref = O.run_mp(T, U0, core, 3)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        fits = t.mp_sweep(3)
        G, U, fit = t.core_and_fit()
    np.testing.assert_allclose(fits, ref["fits"], atol=1e-5)
    for n in range(3):
        assert O.projector_distance(U[n], ref["U"][n]) < 1e-4, n
        assert np.abs(U[n].astype(np.float64).T @ U[n] - np.eye(core[n])).max() < 1e-5


def test_sparse_sp_parity(capi, monkeypatch):
    monkeypatch.setenv("TUCKER_MP_SPARSE", "1")
    from synth import sp_random_init
    dims, nnz, core = (60, 70, 50), 8_000, (6, 7, 5)
    idx, vals, U0 = case(dims, nnz, core)
    T = O.SparseTensor(dims, idx, vals)
    C0 = sp_random_init(dims[2], core[2], np.random.default_rng(3))
    Uinit = [np.zeros((d, j)) for d, j in zip(dims, core)]
    Uinit[2] = C0
    ref = O.run_sp(T, Uinit, core, 3)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        t.set_factor(2, C0.astype(np.float32), check=False)
        fits, _, _ = t.sp_sweep(3)
        _, U, _ = t.core_and_fit()
    np.testing.assert_allclose(fits, ref["fits"], atol=1e-5)
    for n in range(3):
        assert O.projector_distance(U[n], ref["U"][n]) < 1e-4


def test_sparse_mp_deterministic(capi, monkeypatch):
    monkeypatch.setenv("TUCKER_MP_SPARSE", "1")
    dims, nnz, core = (300, 280, 12), 30_000, (9, 7, 5)
    idx, vals, U0 = case(dims, nnz, core)
    out = []
    for _ in range(2):
        with capi.Tucker(dims, core, idx, vals, U0) as t:
            t.mp_sweep(2)
            out.append(t.core_and_fit())
    assert out[0][2] == out[1][2]
    for a, b in zip(out[0][1], out[1][1]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("d,J,gap", [(300, 50, 1e-2), (700, 100, 3e-3), (2000, 60, 1e-2)])
def test_large_eigensolver_parity(capi, monkeypatch, d, J, gap):
    """eig_large on an outlier + flat-bulk spectrum like MP's M_n."""
    monkeypatch.setenv("TUCKER_EIG_LARGE", "1")
    rng = np.random.default_rng(d + J)
    Q = np.linalg.qr(rng.standard_normal((d, d)))[0]
    w = np.sort(rng.uniform(0.1, 1.0, d))[::-1].copy()
    w[0] = 300.0
    w[J - 1] = w[J] * (1 + gap)
    w[:J] = np.maximum(w[:J], w[J - 1])
    S = (Q * w) @ Q.T
    dims, core = (8, 8, 8), (2, 2, 2)
    idx, vals, U0 = case(dims, 50, core)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        U, ev, rc = t.debug_eig(S, J)
    Uo, wo = O.leading_eigenvectors(S, J)
    assert rc == 0
    assert O.projector_distance(U, Uo) < 1e-5
    np.testing.assert_allclose(ev, wo[:J], rtol=1e-9)


def test_core_sizes_above_112(capi):
    """J_n > 112 (the paper's Table 2 cores go to 200^3): the host-driven eigensolver with
    the Rayleigh-Ritz problem on the direct dense solver and SVQB orthonormalisation
    (k > 116), and the tcgen05 SpTTMc in 128-column windows (J_mid, J_leaf > 128).
    HOOI and MP sweeps vs the oracle."""
    from oracle import tucker_oracle as O
    dims, nnz, core = (260, 250, 240), 300_000, (130, 125, 120)
    idx, vals, U0 = case(dims, nnz, core, seed=23, fseed=24)
    T = O.SparseTensor(dims, idx, vals)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        for n in range(3):
            assert O.rel_frobenius(t.debug_ttmc(n), O.ttm_chain_unfold(T, U0, n)) < 1e-4, n
        fh = t.hooi_sweep(2)
        _, Uh, _ = t.core_and_fit()
        t.set_factors(U0)
        fm = t.mp_sweep(2)
        _, Um, _ = t.core_and_fit()
    rh, rm = O.run_hooi(T, U0, core, 2), O.run_mp(T, U0, core, 2)
    np.testing.assert_allclose(fh, rh["fits"], atol=1e-5)
    np.testing.assert_allclose(fm, rm["fits"], atol=1e-5)
    for n in range(3):
        assert O.projector_distance(Uh[n], rh["U"][n]) < 1e-4, ("hooi", n)
        assert O.projector_distance(Um[n], rm["U"][n]) < 1e-4, ("mp", n)


@pytest.mark.parametrize("d,J", [(500, 150), (1200, 200)])
def test_eig_wide_block(capi, d, J):
    rng = np.random.default_rng(d + J)
    Q = np.linalg.qr(rng.standard_normal((d, d)))[0]
    w = np.sort(rng.uniform(0.1, 1.0, d))[::-1].copy()
    w[0] = 80.0
    w[:J] += 0.3
    S = (Q * w) @ Q.T
    dims, core = (8, 8, 8), (2, 2, 2)
    idx, vals, U0 = case(dims, 50, core)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        U, ev, rc = t.debug_eig(S, J)
    Uo, wo = O.leading_eigenvectors(S, J)
    assert rc == 0
    assert O.projector_distance(U, Uo) < 1e-5
    np.testing.assert_allclose(ev, wo[:J], rtol=1e-9)
