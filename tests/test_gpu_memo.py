"""GPU parity of HOOI's partial-contraction reuse at order 4 (DESIGN "HOOI reuse of Z").

Mode p's projection on the ordering (p; p + 1; x; y) keeps Z_v = X x_x U_x^T x_y U_y^T per
node v = (i_p, i_{p+1}); mode p + 1 is then Y_(p+1)[i_{p+1}] = sum_{i_p} U_p[i_p] (x) Z_v
(Fig. 4, Eq. 1 P:274-277 applied in another order).  Checked here: the layout
really pairs the modes, Y of every mode against the oracle through both kernels, stale Z is
never used after a factor changes, whole sweeps against the oracle and against the library
with the reuse switched off, and bit determinism.
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


def case(dims, nnz, core, seed=11, fseed=12):
    rng = np.random.default_rng(seed)
    idx, vals = uniform_distinct_coo(dims, nnz, rng)
    frng = np.random.default_rng(fseed)
    U0 = [random_orthonormal(I, J, frng) for I, J in zip(dims, core)]
    return idx, vals, U0


# dense enough in the mid1 index for the default dispatch to pick the GEMM-form kernel
DENSE = [
    ((24, 20, 32, 18), 33_000, (5, 3, 6, 4)),     # ~12 % dense
    ((40, 33, 20, 35), 90_000, (18, 5, 7, 3)),    # J_root > 16: two U_p column tiles; J_leaf padded to 4
    ((13, 50, 37, 9), 40_000, (4, 20, 3, 6)),     # ragged, J of the sibling mode 20
]


def memo_active(t):
    from paper_0711_2023_b200 import capi as c
    lay = c.tucker_csf_layout(t.h, 4)
    return lay[0]["mid0"] == 1 and lay[2]["mid0"] == 3


@pytest.mark.parametrize("dims,nnz,core", DENSE)
def test_memo_y_parity(capi, dims, nnz, core):
    idx, vals, U0 = case(dims, nnz, core)
    T = O.SparseTensor(dims, idx, vals)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        assert memo_active(t)
        # modes in sweep order: 1 and 3 come from the Z kept by 0 and 2
        Y = [t.debug_ttmc(n) for n in range(4)]
        for n in range(4):
            assert O.rel_frobenius(Y[n], O.ttm_chain_unfold(T, U0, n)) < 1e-4, n
        # a changed factor makes the kept Z stale: new U_2 (a contracted mode of pair (0, 1)),
        # then mode 1 alone must not reuse the old Z
        frng = np.random.default_rng(99)
        U1 = list(U0)
        U1[2] = random_orthonormal(dims[2], core[2], frng)
        t.set_factor(2, U1[2])
        assert O.rel_frobenius(t.debug_ttmc(1), O.ttm_chain_unfold(T, U1, 1)) < 1e-4
        # and a changed U_0 (not contracted in Z of pair (0, 1)) is picked up by the sibling kernel
        t.debug_ttmc(0)
        U1[0] = random_orthonormal(dims[0], core[0], frng)
        t.set_factor(0, U1[0])
        assert O.rel_frobenius(t.debug_ttmc(1), O.ttm_chain_unfold(T, U1, 1)) < 1e-4
        # bit determinism of the sibling kernel
        np.testing.assert_array_equal(t.debug_ttmc(1), t.debug_ttmc(1))


@pytest.mark.parametrize("dims,nnz,core", DENSE)
def test_memo_sweeps(capi, monkeypatch, dims, nnz, core):
    idx, vals, U0 = case(dims, nnz, core)
    T = O.SparseTensor(dims, idx, vals)
    ref = O.run_hooi(T, U0, core, 3)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        assert memo_active(t)
        fits = t.hooi_sweep(3)
        G, U, fit = t.core_and_fit()
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        fits2 = t.hooi_sweep(3)
        _, U2, _ = t.core_and_fit()
    np.testing.assert_array_equal(fits, fits2)
    for n in range(4):
        np.testing.assert_array_equal(U[n], U2[n])
        assert O.projector_distance(U[n], ref["U"][n]) < 1e-4, n
    np.testing.assert_allclose(fits, ref["fits"], atol=1e-5)
    assert abs(fit - ref["fit"]) < 1e-5
    monkeypatch.setenv("TUCKER_HOOI_MEMO", "0")
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        assert not memo_active(t)
        fits0 = t.hooi_sweep(3)
        _, Un, _ = t.core_and_fit()
    np.testing.assert_allclose(fits, fits0, atol=2e-6)
    for n in range(4):
        assert O.projector_distance(U[n], Un[n]) < 1e-4


def test_memo_off_when_sparse(capi):
    """Nodes sparse in the mid1 index: the node-per-warp kernel runs and nothing is kept."""
    dims, nnz, core = (20, 22, 18, 16), 3_000, (4, 5, 3, 6)
    idx, vals, U0 = case(dims, nnz, core)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        assert not memo_active(t)


def test_mp_overlap_times(capi):
    """tucker_mp_overlap_times: counts follow the overlap's structure (order 4, d <= 208: the one-CTA
    solver beside the side stream) -- per sweep N solves and N main-stream Grams, N (N - 1) SpMM terms
    split between the side and main streams -- and every counted time is positive; reset zeroes them."""
    dims, nnz, core = (24, 20, 32, 18), 33_000, (5, 3, 6, 4)
    idx, vals, U0 = case(dims, nnz, core)
    N, S = 4, 3
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        t.mp_sweep(S)
        ov = capi.tucker_mp_overlap_times(t.h)
        assert ov["eig"][1] == N * S and ov["main_gram"][1] == N * S
        # sweep 0 mode 0 builds all N - 1 terms on the main stream; every other mode only the late term
        assert ov["main_spmm"][1] == (N - 1) + (N * S - 1)
        # the side work of the call's last mode is never launched; all others have finished by a sweep's end
        # except possibly the one prepared for the next sweep's first mode (counted only if finished)
        assert N * S - 1 - (S - 1) <= ov["side_gram"][1] <= N * S - 1
        assert ov["side_spmm"][1] == ov["side_gram"][1] * (N - 2)
        for k, (ms, cnt) in ov.items():
            assert ms > 0 and cnt > 0, k
        capi.tucker_mp_overlap_times(t.h, reset=True)
        ov = capi.tucker_mp_overlap_times(t.h)
        assert all(ms == 0 and cnt == 0 for ms, cnt in ov.values())
