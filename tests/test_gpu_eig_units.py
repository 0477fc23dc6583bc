"""GPU unit tests of the fused eigensolver's device routines (through the C-ABI's
debug entry points, include/tucker.h) against plain numpy fp64 definitions:

  - CholQR factor (cholqr_factor, two elimination steps per barrier): M with
    M^T G M = I and M upper triangular with a positive diagonal is unique,
    M = R^{-1} for the upper Cholesky factor R of G (G = R^T R);
  - Jacobi Rayleigh-Ritz eigensolver: eigenvalues vs numpy.linalg.eigvalsh,
    orthonormal V, residual H V - V diag(theta);
  - the split-K DMMA product alpha S Y + gamma D.

Every k from 1 to the build's block limit is covered for CholQR, so both
parities of k - 1 (the trailing single step) and the deferred-row update run.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

K_MAX = 116  # kMaxBlock (internal.cuh)


@pytest.fixture(scope="module")
def capi():
    import __graft_entry__
    __graft_entry__.build()
    from paper_0711_2023_b200 import capi as c
    return c


def spd(k, cond, rng):
    Q = np.linalg.qr(rng.standard_normal((k, k)))[0]
    lam = np.geomspace(1.0, 1.0 / cond, k) * rng.uniform(0.5, 2.0)
    D = np.diag(rng.uniform(0.1, 10.0, k))  # unequal scales: exercises the equilibration
    return D @ (Q * lam) @ Q.T @ D


@pytest.mark.parametrize("k", list(range(1, K_MAX + 1)))
def test_cholqr_factor_equals_inverse_cholesky(capi, k):
    rng = np.random.default_rng(1000 + k)
    for cond in (1e2, 1e8):
        G = spd(k, cond, rng)
        M = capi.tucker_debug_smalldense(0, G, shift=0.0)
        assert np.all(np.tril(M, -1) == 0.0), "M must be upper triangular"
        R = np.linalg.cholesky(G).T  # G = R^T R, R upper
        Mref = np.linalg.inv(R)
        # forward error of a Cholesky-based inverse ~ cond(G) eps
        tol = 50 * cond * 1.1e-16 * max(k, 4)
        err = np.max(np.abs(M - Mref)) / np.max(np.abs(Mref))
        assert err < tol, (k, cond, err)
        orth = np.max(np.abs(M.T @ G @ M - np.eye(k)))
        assert orth < tol, (k, cond, orth)


@pytest.mark.parametrize("k", [2, 3, 9, 40, 59, 60, 61, 82, 115, 116])
def test_jacobi_eigensolver(capi, k):
    rng = np.random.default_rng(2000 + k)
    Q = np.linalg.qr(rng.standard_normal((k, k)))[0]
    lam = np.sort(rng.uniform(1.0, 2.0, k))[::-1]
    lam[: k // 3] += 5.0  # a separated top group plus a cluster
    H = (Q * lam) @ Q.T
    H = 0.5 * (H + H.T)
    V, th, used = capi.tucker_debug_smalldense(1, H, max_sweeps=30)
    assert used > 0
    ref = np.sort(np.linalg.eigvalsh(H))[::-1]
    assert np.max(np.abs(th - ref)) / ref[0] < 1e-12, k
    assert np.all(np.diff(th) <= 0), "descending order"
    assert np.max(np.abs(V.T @ V - np.eye(k))) < 1e-12
    assert np.max(np.abs(H @ V - V * th)) / ref[0] < 1e-11


@pytest.mark.parametrize("d,n", [(1, 1), (7, 3), (100, 60), (257, 61), (1000, 60), (1001, 116), (3000, 8)])
def test_split_k_product(capi, d, n):
    rng = np.random.default_rng(d * 131 + n)
    S = rng.standard_normal((d, d))
    S = S + S.T
    Y = rng.standard_normal((d, n))
    D = rng.standard_normal((d, n))
    out = capi.tucker_debug_product(S, Y, alpha=0.75, gamma=-1.25, D=D)
    ref = 0.75 * (S @ Y) - 1.25 * D
    scale = np.abs(S).sum(axis=1).max() * np.abs(Y).max() + np.abs(D).max()
    assert np.max(np.abs(out - ref)) / scale < 1e-14 * max(d, 16), (d, n)
    out0 = capi.tucker_debug_product(S, Y)
    assert np.max(np.abs(out0 - S @ Y)) / scale < 1e-14 * max(d, 16)


@pytest.mark.parametrize("path", ["auto", "cluster", "packed"])
@pytest.mark.parametrize("d,J,kind", [(3, 1, "spread"), (17, 5, "spread"), (100, 10, "outlier"), (200, 20, "outlier"),
                                      (256, 112, "outlier"), (200, 50, "repeated"), (150, 30, "clustered"),
                                      (210, 25, "repeated"), (64, 64, "spread"), (16, 4, "spread"), (33, 8, "outlier"),
                                      (208, 20, "outlier"), (207, 30, "spread"), (129, 16, "diag"), (200, 20, "diag")])
def test_small_dense_eigensolver(monkeypatch, d, J, kind, path):
    """eig_small against LAPACK: eigenvalues to 1e-12 relative to ||S||, the leading-J
    subspace to 1e-9, orthonormal vectors -- including eigenvalues repeated inside the
    leading set and a tight cluster around the J / J+1 boundary.  "auto": the one-CTA
    solver (k_eig_direct: packed S in shared memory) wherever it fits (d <= 224 and
    the workspace), the 4-CTA cluster path beyond; "cluster": the cluster path forced."""
    if path == "cluster":
        monkeypatch.setenv("TUCKER_EIG_CLUSTER", "1")
    from oracle import tucker_oracle as O
    from paper_0711_2023_b200 import capi
    from synth import random_orthonormal, uniform_distinct_coo
    monkeypatch.setenv("TUCKER_EIG_SMALL", "1")  # the direct solver (experiments; not the default path)
    rng = np.random.default_rng(d + 7 * J)
    Q = np.linalg.qr(rng.standard_normal((d, d)))[0]
    w = np.sort(rng.uniform(0.1, 1.0, d))[::-1].copy()
    if kind == "outlier":
        w[0] = 60.0
    elif kind == "repeated":
        w[:J] = np.repeat(np.linspace(5.0, 2.0, J // 5), 5)  # 5-fold eigenvalues, gap to J+1
    elif kind == "clustered":
        w[:J + 5] = 1.0 + 1e-4 * np.arange(J + 5)[::-1]        # relative gaps 1e-4
        w = np.sort(w)[::-1]
    S = (Q * w) @ Q.T if kind != "diag" else np.diag(rng.permutation(w))
    dims, core = (8, 8, 8), (2, 2, 2)
    idx, vals = uniform_distinct_coo(dims, 50, np.random.default_rng(1))
    U0 = [random_orthonormal(I, c, np.random.default_rng(2)) for I, c in zip(dims, core)]
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        U, ev, rc = t.debug_eig(S, J)
    Uo, wo = O.leading_eigenvectors(S, J)
    assert rc == 0
    np.testing.assert_allclose(ev, wo[:J], rtol=0, atol=1e-12 * wo[0])
    assert np.abs(U.astype(np.float64).T @ U - np.eye(J)).max() < 1e-6
    tol = 1e-9 if kind != "clustered" else 1e-5  # fp32 factor output; clustered: gap 1e-4
    assert O.projector_distance(U, Uo) < max(tol, 1e-6)
