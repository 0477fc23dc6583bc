"""Pins that fix the fp64 oracle to facts outside itself.

Every test here runs on CPU (no GPU marker).  None compares the oracle with
itself: each checks it against a worked example, a closed form, a brute-force
loop, a library routine for a special case, or an invariant of the mathematics.
"""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import tucker_oracle as O
from synth import bernoulli_dense, sp_random_init


def rng(s=0):
    return np.random.default_rng(s)


def rand_sparse(dims, density, seed):
    r = rng(seed)
    X = np.where(r.random(dims) < density, 1.0 - r.random(dims), 0.0)
    return X, O.SparseTensor.from_dense(X)


def rand_factors(dims, core, seed):
    r = rng(seed)
    return [np.linalg.qr(r.standard_normal((I, J)))[0] for I, J in zip(dims, core)]


# ---------------------------------------------------------------- notation --

def test_unfold_matches_eq3_fiber_enumeration():
    # Eq. 3: X_(1) = [x_:11 x_:21 ... x_:I2I3]; Eq. 5: X_(2) = [x_1:1 x_2:1 ...]
    X = np.arange(1, 25, dtype=float).reshape(2, 3, 4)
    X1 = O.unfold(X, 0)
    cols = [X[:, j, k] for k in range(4) for j in range(3)]  # j fastest
    np.testing.assert_array_equal(X1, np.stack(cols, axis=1))
    X2 = O.unfold(X, 1)
    cols = [X[i, :, k] for k in range(4) for i in range(2)]  # i fastest
    np.testing.assert_array_equal(X2, np.stack(cols, axis=1))
    X3 = O.unfold(X, 2)
    cols = [X[i, j, :] for j in range(3) for i in range(2)]
    np.testing.assert_array_equal(X3, np.stack(cols, axis=1))
    for n in range(3):
        np.testing.assert_array_equal(O.fold(O.unfold(X, n), n, X.shape), X)


def test_norm_golden(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "spec_examples.json")))["norm_1_to_8"]
    X = np.arange(1, 9, dtype=float).reshape(g["dims"])
    T = O.SparseTensor.from_dense(X)
    assert T.norm2() == g["value_squared"]


def test_ttm_golden_and_eq1_bruteforce(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "spec_examples.json")))["ttm_all_ones"]
    Y = O.ttm(np.ones(g["dims"]), np.array(g["A"], dtype=float), g["mode"] - 1)
    assert Y.shape == (1, 2, 2) and np.all(Y == g["value"])
    # Eq. 1 with explicit loops
    r = rng(1)
    X = r.standard_normal((3, 4, 5))
    A = r.standard_normal((2, 4))
    Y = O.ttm(X, A, 1)
    Yb = np.zeros((3, 2, 5))
    for i, j, k, l in itertools.product(range(3), range(2), range(5), range(4)):
        Yb[i, j, k] += X[i, l, k] * A[j, l]
    np.testing.assert_allclose(Y, Yb, rtol=1e-13, atol=1e-13)


def test_eq2_matrix_product_as_mode_product():
    # Eq. 2: AB = A x_2 B^T = B x_1 A
    r = rng(2)
    A, B = r.standard_normal((3, 4)), r.standard_normal((4, 5))
    np.testing.assert_allclose(O.ttm(A, B.T, 1), A @ B, rtol=1e-13)
    np.testing.assert_allclose(O.ttm(B, A, 0), A @ B, rtol=1e-13)


def test_tucker_operator_order2_is_usvt():
    # for order 2, [[S; U, V]] = U S V^T
    r = rng(3)
    S, U, V = r.standard_normal((3, 2)), r.standard_normal((5, 3)), r.standard_normal((4, 2))
    np.testing.assert_allclose(O.tucker_operator(S, [U, V]), U @ S @ V.T, rtol=1e-12)


def test_fit_definition_cases():
    # Eq. 9 and the sentence after it
    X = rng(4).standard_normal((3, 4, 5))
    assert O.fit_dense(X, X) == 1.0
    assert abs(O.fit_dense(X, np.zeros_like(X))) < 1e-15
    assert abs(O.fit_dense(X, -X) + 1.0) < 1e-15


# ------------------------------------------------------ P8: SpTTMc chain ----

@pytest.mark.parametrize("dims,core", [((4, 5, 6), (2, 3, 2)), ((3, 4, 2, 5), (2, 2, 2, 3))])
def test_ttm_chain_bruteforce_loops(dims, core):
    X, T = rand_sparse(dims, 0.4, 5)
    U = rand_factors(dims, core, 6)
    N = len(dims)
    for n in range(N):
        Y = O.ttm_chain_unfold(T, U, n)
        others = [m for m in range(N) if m != n]
        P = int(np.prod([core[m] for m in others]))
        Yb = np.zeros((dims[n], P))
        # pure loops over nonzeros and output columns, Eq. 1 applied N-1 times;
        # Kolda column index: lower modes fastest
        for e in range(T.vals.size):
            ii = [T.idx[m][e] for m in range(N)]
            for js in itertools.product(*[range(core[m]) for m in others]):
                col, stride = 0, 1
                prod = T.vals[e]
                for m, j in zip(others, js):
                    col += j * stride
                    stride *= core[m]
                    prod *= U[m][ii[m], j]
                Yb[ii[n], col] += prod
        np.testing.assert_allclose(Y, Yb, rtol=1e-12, atol=1e-12)


def test_ttm_chain_kronecker_law():
    # P:319-321 applied N-1 times: Y_(n) = X_(n) (U_N x ... x U_1 without n)
    dims, core = (6, 7, 5), (3, 2, 4)
    X, T = rand_sparse(dims, 0.3, 7)
    U = rand_factors(dims, core, 8)
    for n in range(3):
        others = [m for m in range(3) if m != n]
        K = np.kron(U[others[1]], U[others[0]])  # later mode slower -> left factor
        np.testing.assert_allclose(O.ttm_chain_unfold(T, U, n), O.unfold(X, n) @ K, rtol=1e-12, atol=1e-13)


# ---------------------------------------------------------- eigenvectors ----

def test_leading_eigenvectors_golden(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "spec_examples.json")))["eig_2x2"]
    V, w = O.leading_eigenvectors(np.array(g["S"], dtype=float), 2)
    np.testing.assert_allclose(w, g["eigenvalues"], rtol=1e-14)
    np.testing.assert_allclose(V, np.array(g["eigenvectors_cols"]), atol=1e-14)
    V, _ = O.leading_eigenvectors(np.diag([4.0, 1.0]), 1)
    np.testing.assert_array_equal(V[:, 0], [1.0, 0.0])


def test_leading_eigenvectors_vs_power_deflation():
    # independent oracle: power iteration with deflation (S:140 third example)
    r = rng(9)
    B = r.standard_normal((6, 6))
    S = B @ B.T + np.diag([30.0, 20, 10, 0, 0, 0])
    V, w = O.leading_eigenvectors(S, 3)
    R = S.copy()
    for j in range(3):
        v = np.ones(6)
        for _ in range(5000):
            v = R @ v
            v /= np.linalg.norm(v)
        lam = v @ R @ v
        assert abs(abs(v @ V[:, j]) - 1) < 1e-9
        assert abs(lam - w[j]) < 1e-9 * abs(w[0])
        R = R - lam * np.outer(v, v)
    assert np.linalg.norm(S @ V - V * w[:3]) < 1e-10 * np.linalg.norm(S)


# ------------------------------------------------------------- P1 / P2 ----

@pytest.mark.parametrize("algo", ["hooi", "mp"])
@pytest.mark.parametrize("dims,core", [((8, 9, 10), (2, 3, 2)), ((5, 6, 4, 5), (2, 2, 3, 2))])
def test_p1_exact_multilinear_rank_fit_one(algo, dims, core):
    r = rng(10)
    C = r.standard_normal(core)
    A = [np.linalg.qr(r.standard_normal((I, J)))[0] for I, J in zip(dims, core)]
    X = O.tucker_operator(C, A)
    T = O.SparseTensor.from_dense(X)
    U0 = rand_factors(dims, core, 11)
    run = O.run_hooi if algo == "hooi" else O.run_mp
    out = run(T, U0, core, 1)
    assert out["fit"] > 1 - 1e-6
    for n in range(len(dims)):
        assert O.projector_distance(out["U"][n], A[n]) < 1e-8


def test_p2_full_core_reconstructs():
    dims = (4, 5, 3)
    X, T = rand_sparse(dims, 0.5, 12)
    U = rand_factors(dims, dims, 13)  # square orthogonal factors
    G = O.core(T, U)
    np.testing.assert_allclose(O.tucker_operator(G, U), X, atol=1e-12)
    assert abs(O.fit_from_core(T.norm2(), G) - 1.0) < 1e-6
    assert abs(O.fit_residual(T, G, U) - 1.0) < 1e-12


# ------------------------------------------------------ P3 / P7 / P10 ----

def test_p3_p7_p10_hooi_properties():
    dims, core = (12, 10, 14), (3, 4, 2)
    X, T = rand_sparse(dims, 0.3, 14)
    U = rand_factors(dims, core, 15)
    nx2 = T.norm2()
    prev = -np.inf
    for _ in range(4):
        Uw = [u.copy() for u in U]
        for n in range(3):  # P10: ||G|| non-decreasing after every mode update
            Y = O.ttm_chain_unfold(T, Uw, n)
            Uw[n], _ = O.leading_eigenvectors(Y @ Y.T, core[n])
            g = np.linalg.norm(Uw[n].T @ Y)
            assert g >= prev - 1e-12 * np.sqrt(nx2)
            prev = g
        U = Uw
        for u in U:  # P3
            assert np.abs(u.T @ u - np.eye(u.shape[1])).max() < 1e-12
        G = O.core(T, U)
        # P7: norm identity equals the dense residual (Eq. 9)
        assert abs(O.fit_from_core(nx2, G) - O.fit_residual(T, G, U)) < 1e-12


# ------------------------------------------------------------------- P4 ----

def test_p4_order2_hooi_is_truncated_svd_and_mp_equals_hooi_gram():
    X, T = rand_sparse((30, 20), 0.4, 16)
    core = (4, 4)
    U0 = rand_factors((30, 20), core, 17)
    out = O.run_hooi(T, U0, core, 400)  # sigma_4/sigma_5 = 1.03: slow alternating convergence
    Us, s, Vt = np.linalg.svd(X)
    fit_svd = 1 - np.sqrt(np.sum(s[4:] ** 2)) / np.linalg.norm(s)
    assert abs(out["fit"] - fit_svd) < 1e-9
    assert O.projector_distance(out["U"][0], Us[:, :4]) < 1e-6
    assert O.projector_distance(out["U"][1], Vt[:4].T) < 1e-6
    # MP for order 2: M_1 is the single term (X x_2 U2^T)_(1)(.)^T = Y_(1) Y_(1)^T
    Y = O.ttm_chain_unfold(T, U0, 0)
    np.testing.assert_allclose(O.mp_gram(T, U0, 0), Y @ Y.T, rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------- P5 / P6 ----

def test_p5_hosvd_equals_svd_of_unfolding():
    dims, core = (6, 7, 8), (3, 2, 4)
    X, T = rand_sparse(dims, 0.6, 18)
    for n in range(3):
        Un = O.hosvd_factor(T, n, core[n])
        Us = np.linalg.svd(O.unfold(X, n))[0][:, :core[n]]
        assert O.projector_distance(Un, Us) < 1e-10


@pytest.mark.parametrize("dims", [(6, 7, 8), (4, 5, 3, 6)])
def test_p6_pseudo_hosvd_is_multiple_of_xxT(dims):
    X, T = rand_sparse(dims, 0.5, 19)
    N = len(dims)
    for n in range(N):
        Xn = O.unfold(X, n)
        np.testing.assert_allclose(O.pseudo_hosvd_gram(T, n), (N - 1) * Xn @ Xn.T, rtol=1e-12)


# ------------------------------------------------------------------- P9 ----

@pytest.mark.parametrize("dims,core", [((5, 4, 6), (2, 3, 2)), ((4, 3, 5, 3), (2, 2, 3, 2))])
def test_p9_mp_gram_slice_loop_and_bruteforce(dims, core):
    X, T = rand_sparse(dims, 0.5, 20)
    U = rand_factors(dims, core, 21)
    N = len(dims)
    for n in range(N):
        M = O.mp_gram(T, U, n)
        np.testing.assert_allclose(M, O.mp_gram_slices(T, U, n), rtol=1e-12, atol=1e-12)
        # brute force from the dense X: M[a,b] = sum_{m!=n} sum_{fixed idx} sum_j p_a p_b,
        # p_a = sum_{i_m} x[..a..i_m..] U_m[i_m, j]
        Mb = np.zeros((dims[n], dims[n]))
        for m in range(N):
            if m == n:
                continue
            fixed = [k for k in range(N) if k not in (n, m)]
            for fix in itertools.product(*[range(dims[k]) for k in fixed]):
                for j in range(core[m]):
                    p = np.zeros(dims[n])
                    for a in range(dims[n]):
                        for im in range(dims[m]):
                            ix = [0] * N
                            ix[n], ix[m] = a, im
                            for k, v in zip(fixed, fix):
                                ix[k] = v
                            p[a] += X[tuple(ix)] * U[m][im, j]
                    Mb += np.outer(p, p)
        np.testing.assert_allclose(M, Mb, rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------ P11 ----

def test_p11_permutation_and_scaling_invariance():
    dims, core = (9, 8, 7), (3, 2, 3)
    X, T = rand_sparse(dims, 0.4, 22)
    U0 = rand_factors(dims, core, 23)
    base = O.run_hooi(T, U0, core, 3)
    perm = rng(24).permutation(dims[1])
    Xp = X[:, perm, :]
    U0p = [U0[0], U0[1][perm], U0[2]]
    outp = O.run_hooi(O.SparseTensor.from_dense(Xp), U0p, core, 3)
    assert abs(outp["fit"] - base["fit"]) < 1e-12
    assert O.projector_distance(outp["U"][1], base["U"][1][perm]) < 1e-9
    outs = O.run_hooi(O.SparseTensor.from_dense(3.5 * X), U0, core, 3)
    assert abs(outs["fit"] - base["fit"]) < 1e-12
    for n in range(3):
        assert O.projector_distance(outs["U"][n], base["U"][n]) < 1e-9


# ------------------------------------------------------------------ P13 ----

def test_p13_sharded_gram_sum_equals_full():
    dims, core = (40, 12, 11), (4, 3, 3)
    X, T = rand_sparse(dims, 0.3, 25)
    U = rand_factors(dims, core, 26)
    Y = O.ttm_chain_unfold(T, U, 0)
    bounds = [0, 13, 27, 40]  # row-owner shards by mode-n index range (§8(e))
    S = sum(Y[a:b].T @ Y[a:b] for a, b in zip(bounds[:-1], bounds[1:]))
    np.testing.assert_allclose(S, Y.T @ Y, rtol=1e-13, atol=1e-13)
    M = O.mp_gram(T, U, 1)
    parts = []
    for a, b in zip(bounds[:-1], bounds[1:]):  # MP: shard by slice-mode index
        sel = (T.idx[0] >= a) & (T.idx[0] < b)
        Ts = O.SparseTensor(dims, [i[sel] for i in T.idx], T.vals[sel])
        parts.append(Ts)
    # term m=2 slices fix mode 0, term m=0 slices fix mode 2 -> shard each term by its slice mode
    W2 = sum((lambda W: W @ W.T)(O.mp_term_unfold(Ts, U[2], 1, 2)) for Ts in parts)
    W0 = O.mp_term_unfold(T, U[0], 1, 0)
    np.testing.assert_allclose(W2 + W0 @ W0.T, M, rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------ P12 ----

def _paper_fit_case(golden_dir, key, seed):
    g = json.load(open(os.path.join(golden_dir, "paper_fits.json")))
    case, tol = g[key], g["tolerance_pp"]
    X = bernoulli_dense(tuple(case["dims"]), case["density"], np.random.default_rng(seed))
    return O.SparseTensor.from_dense(X), case, tol


@pytest.mark.slow
def test_p12_table2_statistical_pin(golden_dir):
    T, case, tol = _paper_fit_case(golden_dir, "table2_250cube_J25", 1)
    core = tuple(case["core"])
    assert abs(100 * O.run_hosvd(T, core)["fit"] - case["hosvd"]) < tol
    assert abs(100 * O.run_hooi_converged(T, core)["fit"] - case["hooi"]) < tol
    assert abs(100 * O.run_mp_converged(T, core)["fit"] - case["mp"]) < tol


@pytest.mark.slow
def test_p12_table6_statistical_pin(golden_dir):
    T, case, tol = _paper_fit_case(golden_dir, "table6_100pow4_J20", 1)
    core = tuple(case["core"])
    assert abs(100 * O.run_hooi_converged(T, core)["fit"] - case["hooi"]) < tol
    assert abs(100 * O.run_mp_converged(T, core)["fit"] - case["mp"]) < tol


# ------------------------------------------------------ Slice Projection ----
# Figs. 5-6 written out literally with dense slices, against the
# oracle's sp_gram (which reuses MP's single-term unfolding): pins the mode
# mapping (mode n from the previous mode's factor, slices on the remaining
# modes) against the figures themselves.

def test_sp_gram_matches_figure5_slice_loops():
    rng = np.random.default_rng(71)
    I1, I2, I3 = 5, 6, 7
    X = rng.random((I1, I2, I3)) * (rng.random((I1, I2, I3)) < 0.5)
    T = O.SparseTensor.from_dense(X)
    A, B, C = rng.random((I1, 2)), rng.random((I2, 3)), rng.random((I3, 2))
    U = [A, B, C]
    M13 = sum(X[:, i, :] @ C @ C.T @ X[:, i, :].T for i in range(I2))       # slices on mode 2
    M21 = sum(X[:, :, i].T @ A @ A.T @ X[:, :, i] for i in range(I3))       # slices on mode 3
    M32 = sum(X[i, :, :].T @ B @ B.T @ X[i, :, :] for i in range(I1))       # slices on mode 1
    for n, M in enumerate((M13, M21, M32)):
        np.testing.assert_allclose(O.sp_gram(T, U, n), M, rtol=1e-12, atol=1e-12)


def test_sp_gram_matches_figure6_slice_loops():
    rng = np.random.default_rng(72)
    d = (3, 4, 5, 3)
    X = rng.random(d) * (rng.random(d) < 0.6)
    T = O.SparseTensor.from_dense(X)
    A, B, C, D = (rng.random((n, 2)) for n in d)
    U = [A, B, C, D]
    M14 = sum(X[:, i, j, :] @ D @ D.T @ X[:, i, j, :].T for i in range(d[1]) for j in range(d[2]))
    M21 = sum(X[:, :, i, j].T @ A @ A.T @ X[:, :, i, j] for i in range(d[2]) for j in range(d[3]))
    M32 = sum(X[i, :, :, j].T @ B @ B.T @ X[i, :, :, j] for i in range(d[0]) for j in range(d[3]))
    M43 = sum(X[i, j, :, :].T @ C @ C.T @ X[i, j, :, :] for i in range(d[0]) for j in range(d[1]))
    for n, M in enumerate((M14, M21, M32, M43)):
        np.testing.assert_allclose(O.sp_gram(T, U, n), M, rtol=1e-12, atol=1e-12)


def test_sp_exact_multilinear_rank_fit_one():
    rng = np.random.default_rng(73)
    dims, core = (12, 10, 9), (3, 2, 2)
    G = rng.standard_normal(core)
    Us = [np.linalg.qr(rng.standard_normal((I, J)))[0] for I, J in zip(dims, core)]
    X = O.tucker_operator(G, Us)
    T = O.SparseTensor.from_dense(X)
    r = O.run_sp(T, [np.zeros((I, J)) for I, J in zip(dims[:-1], core[:-1])] +
                 [sp_random_init(dims[-1], core[-1], rng)], core, 3)
    # exact rank: the core keeps all of X (||G|| = ||X||); the fit's sqrt turns
    # 1e-16 rounding of ||X||^2 - ||G||^2 into ~1e-8
    assert abs(r["gnorms"][-1] / np.sqrt(T.norm2()) - 1.0) < 1e-12
    assert abs(r["fits"][-1] - 1.0) < 1e-6
    # Delta_G proxy (Eq. 11) is consistent: the core norm never decreases here
    assert np.all(np.diff(r["gnorms"]) > -1e-12)


@pytest.mark.slow
def test_p12_table2_sp_statistical_pin(golden_dir):
    """The paper's SP fit at 250^3 (Table 2: 3.934 %) from a random
    uniform, column-normalised last factor, Delta_G < 1e-4 (Eq. 11)."""
    T, case, tol = _paper_fit_case(golden_dir, "table2_250cube_J25", 1)
    core = tuple(case["core"])
    C0 = sp_random_init(T.dims[-1], core[-1], np.random.default_rng(7))
    assert abs(100 * O.run_sp_converged(T, core, C0)["fit"] - case["sp"]) < tol


# ------------------------------------- the parity metric and the large-tensor routes ----

def test_projector_distance_pins():
    """The metric behind every factor-parity assertion, pinned to its definition
    ||U U^T - V V^T||_F written out with explicit I x I projectors, and to closed
    forms: a subspace that differs in one orthogonal direction is sqrt(2) away,
    orthogonal J-dimensional subspaces are sqrt(2 J) apart, and rotating or
    sign-flipping the basis changes nothing."""
    r = rng(40)
    for I, J in [(7, 1), (12, 3), (30, 5), (9, 9)]:
        U = np.linalg.qr(r.standard_normal((I, J)))[0]
        V = np.linalg.qr(r.standard_normal((I, J)))[0]
        explicit = np.linalg.norm(U @ U.T - V @ V.T)
        assert abs(O.projector_distance(U, V) - explicit) < 1e-12
        Q = np.linalg.qr(r.standard_normal((J, J)))[0]
        assert O.projector_distance(U, U @ Q) < 1e-12
        assert O.projector_distance(U, U * np.where(np.arange(J) % 2, -1.0, 1.0)) < 1e-12
    # one column swapped for a direction orthogonal to the whole subspace
    B = np.linalg.qr(r.standard_normal((10, 4)))[0]
    U, V = B[:, :3], np.c_[B[:, :2], B[:, 3]]
    assert abs(O.projector_distance(U, V) - np.sqrt(2.0)) < 1e-12
    # mutually orthogonal subspaces
    assert abs(O.projector_distance(B[:, :2], B[:, 2:]) - 2.0) < 1e-12
    # small rotation by angle eps out of the subspace: distance = sqrt(2) sin(eps)
    eps = 1e-5
    W = B[:, :3].copy()
    W[:, 0] = np.cos(eps) * B[:, 0] + np.sin(eps) * B[:, 3]
    assert abs(O.projector_distance(B[:, :3], W) - np.sqrt(2.0) * np.sin(eps)) < 1e-15


@pytest.mark.parametrize("dims,core,density", [((7, 9, 5), (2, 3, 2), 0.3), ((11, 4, 6), (3, 2, 4), 0.15),
                                                ((5, 13, 8), (4, 5, 3), 0.05)])
def test_slice_chain_matches_eq1_loops(dims, core, density):
    """ttm_chain_unfold_slices (the Appendix's B' X_slice C per slice) against
    pure Eq. 1 loops over the nonzeros (no shared code), ragged dims and sparse
    enough that some slices and fibers are empty."""
    X, T = rand_sparse(dims, density, 41)
    U = rand_factors(dims, core, 42)
    for n in range(3):
        Y = O.ttm_chain_unfold_slices(T, U, n)
        others = [m for m in range(3) if m != n]
        Yb = np.zeros((dims[n], core[others[0]] * core[others[1]]))
        for e in range(T.vals.size):
            ii = [T.idx[m][e] for m in range(3)]
            for ja in range(core[others[0]]):
                for jb in range(core[others[1]]):
                    Yb[ii[n], ja + core[others[0]] * jb] += (T.vals[e] * U[others[0]][ii[others[0]], ja]
                                                             * U[others[1]][ii[others[1]], jb])
        np.testing.assert_allclose(Y, Yb, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(Y, O.ttm_chain_unfold(T, U, n), rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("shape,J", [((40, 12), 3), ((57, 9), 9), ((25, 24), 5)])
def test_gram_t_route_is_left_singular_subspace(shape, J):
    """Reading A10: U from Y^T Y equals the J leading left singular vectors of Y
    (numpy's SVD, a library routine) and the Y Y^T route, including the sign
    convention; it is orthonormal and its eigenvalues are sigma^2."""
    r = rng(43)
    Y = r.standard_normal(shape) @ np.diag(np.linspace(3.0, 1.0, shape[1]))
    U, w = O.leading_left_vectors_gram_t(Y, J)
    Us, sv, _ = np.linalg.svd(Y, full_matrices=False)
    assert O.projector_distance(U, Us[:, :J]) < 1e-10
    np.testing.assert_allclose(w[:J], sv[:J] ** 2, rtol=1e-12)
    assert np.abs(U.T @ U - np.eye(J)).max() < 1e-12
    V, _ = O.leading_eigenvectors(Y @ Y.T, J)
    np.testing.assert_allclose(U, V, atol=1e-10)  # same columns, same signs
    with pytest.raises(ValueError):
        O.leading_left_vectors_gram_t(np.c_[Y[:, :2], Y[:, :2]], 4)  # rank 2 < J


@pytest.mark.parametrize("dims,core", [((30, 8, 9), (4, 3, 3)), ((10, 12, 40), (3, 4, 5))])
def test_hooi_large_matches_hooi(dims, core):
    """The large-tensor driver (slice-wise chain, Y^T Y route where I_n > prod J,
    core from the last projection) reproduces run_hooi sweep by sweep; both Gram
    routes occur in these shapes."""
    X, T = rand_sparse(dims, 0.2, 44)
    U0 = rand_factors(dims, core, 45)
    assert any(dims[n] > np.prod([core[m] for m in range(3) if m != n]) for n in range(3))
    a = O.run_hooi(T, U0, core, 3)
    b = O.run_hooi_large(T, U0, core, 3)
    np.testing.assert_allclose(b["fits"], a["fits"], atol=1e-12)
    for n in range(3):
        assert O.projector_distance(a["U"][n], b["U"][n]) < 1e-9
    np.testing.assert_allclose(b["G"], O.core(T, b["U"]), atol=1e-12)


def test_hooi_large_exact_multilinear_rank():
    """P1 through the large-tensor driver: exact multilinear rank gives fit 1."""
    dims, core = (40, 9, 10), (3, 2, 4)
    r = rng(46)
    C = r.standard_normal(core)
    A = [np.linalg.qr(r.standard_normal((I, J)))[0] for I, J in zip(dims, core)]
    T = O.SparseTensor.from_dense(O.tucker_operator(C, A))
    out = O.run_hooi_large(T, rand_factors(dims, core, 47), core, 1)
    assert out["fit"] > 1 - 1e-6
    for n in range(3):
        assert O.projector_distance(out["U"][n], A[n]) < 1e-8


@pytest.mark.parametrize("dims,core", [((7, 9, 5), (2, 3, 2)), ((11, 4, 13), (3, 2, 4))])
def test_mp_gram_rows_is_a_row_of_the_slice_loop(dims, core):
    """mp_gram_rows (MP's M_n rows without forming M_n) against the literal Fig. 7 slice
    loop mp_gram_slices (P9), including rows with no nonzero (zero rows)."""
    X, T = rand_sparse(dims, 0.2, 48)
    U = rand_factors(dims, core, 49)
    for n in range(3):
        M = O.mp_gram_slices(T, U, n)
        rows = list(range(dims[n]))
        np.testing.assert_allclose(O.mp_gram_rows(T, U, n, rows), M, rtol=1e-12, atol=1e-12)
        # slices visited in chunks of a few nonzeros: the same rows
        np.testing.assert_allclose(O.mp_gram_rows(T, U, n, rows, chunk=7), M, rtol=1e-12, atol=1e-12)
