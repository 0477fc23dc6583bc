"""fp64 CPU oracle for the HOOI / Multislice-Projection hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product path (``paper_0711_2023_b200`` + ``libtucker.so``) never
imports, links or executes it, and it shares no code with that path.

Every function is a plain restatement of PAPER.md (``P:<line>``) in float64 with
numpy/scipy primitives (sparse x dense product, tensordot, matmul, ``eigh``).
There is no blocking, fusion or reordering beyond what the definitions state.
Readings of ambiguous passages are the SURVEY.md §8(c) ledger entries A1-A18,
restated in DESIGN.md.

Parity status per function:
  unfold, ttm, tucker_operator, fit_dense   pinned (tests/test_oracle_pins.py)
  ttm_chain_unfold                           pinned (brute force P8, Kronecker law)
  leading_eigenvectors                       pinned (SPEC worked examples, residual)
  hooi_sweep / run_hooi                      pinned (P1, P2, P4, P10, P12)
  mp_gram / mp_gram_slices / run_mp          pinned (P1, P4, P6, P9, P12)
  core / fit_from_core                       pinned (P2, P7)
  hosvd, pseudo_hosvd                        pinned (P5, P6, P12)
  ttm_chain_unfold_slices                    pinned (Eq. 1 brute force, = ttm_chain_unfold)
  leading_left_vectors_gram_t                pinned (SVD of Y, = the Y Y^T route, ragged shapes)
  hooi_sweep_large / run_hooi_large          pinned (= hooi_sweep / run_hooi on small tensors,
                                             P1 exact multilinear rank)
  projector_distance                         pinned (explicit ||U U^T - V V^T||_F, sqrt 2 for
                                             one swapped column, rotation/sign invariance)
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

# ---------------------------------------------------------------------------
# Dense notation (§3)
# ---------------------------------------------------------------------------


def unfold(X: np.ndarray, n: int) -> np.ndarray:
    """Mode-n matricization X_(n) (Eqs. 3-6).

    Columns are mode-n fibers, ordered with the lower-numbered remaining modes
    varying fastest (Eq. 3: X_(1) = [x_:11 x_:21 ... x_:I2I3]).  Reading A9
    extends the rule to every mode.  `n` is 0-based here.
    """
    return np.moveaxis(X, n, 0).reshape(X.shape[n], -1, order="F")


def fold(M: np.ndarray, n: int, dims) -> np.ndarray:
    """Inverse of :func:`unfold`."""
    rest = [d for i, d in enumerate(dims) if i != n]
    return np.moveaxis(M.reshape([dims[n]] + rest, order="F"), 0, n)


def ttm(X: np.ndarray, A: np.ndarray, n: int) -> np.ndarray:
    """n-mode product Y = X x_n A, Eq. 1:
    y_{..j..} = sum_{i_n} x_{..i_n..} a_{j i_n}.  Uses Y_(n) = A X_(n)."""
    dims = list(X.shape)
    dims[n] = A.shape[0]
    return fold(A @ unfold(X, n), n, dims)


def tucker_operator(G: np.ndarray, factors) -> np.ndarray:
    """[[G; A1..AN]] = G x_1 A1 x_2 ... x_N AN, Eq. 7."""
    Y = G
    for n, A in enumerate(factors):
        Y = ttm(Y, A, n)
    return Y


def fit_dense(X: np.ndarray, Xhat: np.ndarray) -> float:
    """fit = 1 - ||X - Xhat||_F / ||X||_F, Eq. 9."""
    nx = np.linalg.norm(X.ravel())
    if nx == 0:
        raise ValueError("fit undefined for a zero tensor (S:95)")
    return float(1.0 - np.linalg.norm((X - Xhat).ravel()) / nx)


# ---------------------------------------------------------------------------
# Sparse tensor container (COO: one <i,j,k,x> per nonzero)
# ---------------------------------------------------------------------------


class SparseTensor:
    """Order-N COO tensor in float64 (0-based indices)."""

    def __init__(self, dims, idx, vals):
        self.dims = tuple(int(d) for d in dims)
        self.N = len(self.dims)
        self.idx = [np.asarray(a, dtype=np.int64) for a in idx]
        self.vals = np.asarray(vals, dtype=np.float64)
        assert len(self.idx) == self.N
        keep = self.vals != 0.0  # explicit zeros are dropped
        if not keep.all():
            self.idx = [a[keep] for a in self.idx]
            self.vals = self.vals[keep]

    @classmethod
    def from_dense(cls, X: np.ndarray) -> "SparseTensor":
        nz = np.nonzero(X)
        return cls(X.shape, nz, X[nz])

    def to_dense(self) -> np.ndarray:
        X = np.zeros(self.dims)
        np.add.at(X, tuple(self.idx), self.vals)
        return X

    def norm2(self) -> float:
        """||X||_F^2."""
        return float(np.dot(self.vals, self.vals))

    def matrix(self, rows: list[int], col: int) -> sp.csr_matrix:
        """The sparse matrix whose row is the linear index over `rows` modes
        (lowest mode fastest) and whose column is the index in mode `col`."""
        r = np.zeros_like(self.vals, dtype=np.int64)
        stride = 1
        for m in rows:
            r += self.idx[m] * stride
            stride *= self.dims[m]
        return sp.csr_matrix((self.vals, (r, self.idx[col])), shape=(stride, self.dims[col]))


# ---------------------------------------------------------------------------
# HOOI projection: Z = [[X; A1^T, ..., I_n, ..., AN^T]] (Fig. 4)
# ---------------------------------------------------------------------------


def ttm_chain(T: SparseTensor, U, n: int) -> np.ndarray:
    """Dense tensor Z = X x_{m != n} U_m^T (Fig. 4 `Z <- [[X; A(1)T..I_n..A(N)T]]`).

    Axis m of the result has size J_m for m != n and I_n for m == n.
    The first product is sparse x dense (Eq. 1 over the nonzeros), the rest are
    dense n-mode products (Eq. 1).  Product order is irrelevant mathematically
    (the n-mode products in distinct modes commute); the smallest J goes first
    only to bound memory.
    """
    others = sorted((m for m in range(T.N) if m != n), key=lambda m: U[m].shape[1])
    m0 = others[0]
    rest_modes = [m for m in range(T.N) if m != m0]
    # X x_{m0} U_{m0}^T : rows = linear index over rest_modes (lowest fastest)
    Z = T.matrix(rest_modes, m0) @ np.asarray(U[m0], dtype=np.float64)
    shape_rest = [T.dims[m] for m in rest_modes]
    Z = Z.reshape(shape_rest + [U[m0].shape[1]], order="F")
    # axes currently: rest_modes..., m0 -> move m0 back into its slot
    Z = np.moveaxis(Z, -1, m0)
    for m in others[1:]:
        Z = ttm(Z, np.asarray(U[m], dtype=np.float64).T, m)
    return Z


def ttm_chain_unfold(T: SparseTensor, U, n: int) -> np.ndarray:
    """Y_(n) = Z_(n), I_n x prod_{m != n} J_m, Kolda column order (Eqs. 3-6)."""
    return unfold(ttm_chain(T, U, n), n)


def ttm_chain_unfold_slices(T: SparseTensor, U, n: int) -> np.ndarray:
    """Y_(n) = (X x_{m != n} U_m^T)_(n) for ORDER-3 tensors, one mode-n slice at a
    time, as the paper's own code forms it: row i of Y_(1) is B' * X1_slice * C
    (Appendix) with X1_slice the I_a x I_b slice of index i (a < b the two
    other modes).  That is Eq. 1 applied to the slice twice; only the rows of the
    slice that hold nonzeros (its fibers) take part, so no dense I_a x J_b
    intermediate is formed.  The row is the J_a x J_b matrix U_a^T X_i U_b
    flattened with the lower mode fastest (Kolda order, Eqs. 3-6).  Memory and
    time grow with the nonzeros and fibers only (config 5 of BASELINE.json)."""
    if T.N != 3:
        raise ValueError("ttm_chain_unfold_slices: order 3 only")
    a, b = [m for m in range(3) if m != n]
    Ua = np.asarray(U[a], dtype=np.float64)
    Ub = np.asarray(U[b], dtype=np.float64)
    Ja, Jb = Ua.shape[1], Ub.shape[1]
    Y = np.zeros((T.dims[n], Ja * Jb))
    # the slice / fiber grouping depends on the tensor only: kept on T for later sweeps
    plans = T.__dict__.setdefault("_slice_plans", {})
    if n not in plans:
        i_n, i_a, i_b = T.idx[n], T.idx[a], T.idx[b]
        order = np.lexsort((i_b, i_a, i_n))
        i_n, i_a, i_b, x = i_n[order], i_a[order], i_b[order], T.vals[order]
        # fibers = distinct (i_n, i_a): the nonzero rows of each slice X_i
        fkey = i_n * T.dims[a] + i_a
        fstart = np.flatnonzero(np.r_[True, fkey[1:] != fkey[:-1]])
        del fkey
        f_n, f_a = i_n[fstart], i_a[fstart]
        del i_n, i_a
        sstart = np.flatnonzero(np.r_[True, f_n[1:] != f_n[:-1]])
        plans[n] = (i_b, x, fstart, f_n, f_a, sstart)
    i_b, x, fstart, f_n, f_a, sstart = plans[n]
    send = np.r_[sstart[1:], f_n.size]
    fend_nz = np.r_[fstart[1:], x.size]
    # process slices in chunks of <= ~2e6 fibers: t_f = X_i[row f, :] U_b (Eq. 1)
    s0 = 0
    while s0 < sstart.size:
        s1 = s0 + 1
        while s1 < sstart.size and send[s1] - sstart[s0] <= 2_000_000:
            s1 += 1
        f0, f1 = sstart[s0], send[s1 - 1]
        e0, e1 = fstart[f0], fend_nz[f1 - 1]
        rows = np.repeat(np.arange(f1 - f0), np.diff(np.r_[fstart[f0:f1], e1]))
        Xf = sp.csr_matrix((x[e0:e1], (rows, i_b[e0:e1])), shape=(f1 - f0, T.dims[b]))
        Tf = Xf @ Ub                                    # fibers x J_b
        for s in range(s0, s1):
            g0, g1 = sstart[s] - f0, send[s] - f0
            M = Ua[f_a[sstart[s] : send[s]]].T @ Tf[g0:g1]  # U_a^T X_i U_b (J_a x J_b)
            Y[f_n[sstart[s]]] = M.ravel(order="F")  # j_a + J_a j_b (a < b)
        s0 = s1
    return Y


def leading_eigenvectors(S: np.ndarray, J: int):
    """J leading eigenvectors of symmetric S (Fig. 4 `A(n) <- J_n leading
    eigenvectors of Z_(n) Z_(n)^T`), descending eigenvalue order, each column
    sign-canonicalised (largest-magnitude entry positive, ties -> lowest
    index).  Reading A2: the eigenvectors of M (not of M M^T).
    Returns (U, w_all_descending)."""
    S = np.asarray(S, dtype=np.float64)
    w, V = np.linalg.eigh(0.5 * (S + S.T))
    order = np.argsort(-w, kind="stable")
    w = w[order]
    V = V[:, order[:J]].copy()
    for j in range(V.shape[1]):
        k = int(np.argmax(np.abs(V[:, j])))  # argmax returns lowest index on ties
        if V[k, j] < 0:
            V[:, j] = -V[:, j]
    return V, w


def leading_left_vectors_gram_t(Y: np.ndarray, J: int):
    """The J leading eigenvectors of Y Y^T computed from the smaller Gram Y^T Y
    (reading A10, used when I_n > prod_{m != n} J_m): with Y^T Y = V Theta V^T,
    the left singular vectors are U = Y V Theta^{-1/2} (Y = U Sigma V^T, Theta =
    Sigma^2), orthonormal in exact arithmetic.  Descending order, columns
    sign-canonicalised as in :func:`leading_eigenvectors`.  Returns
    (U, w) with w the eigenvalues of Y^T Y, descending (the nonzero spectrum of
    Y Y^T)."""
    Y = np.asarray(Y, dtype=np.float64)
    if J > Y.shape[1]:
        raise ValueError("Y^T Y route: J exceeds the columns of Y")
    w, V = np.linalg.eigh(Y.T @ Y)
    order = np.argsort(-w, kind="stable")
    w = w[order]
    V = V[:, order[:J]]
    if not w[J - 1] > 1e-12 * w[0]:  # reading A10: theta_J <= 1e-12 theta_1 is rank deficient
        raise ValueError("Y^T Y route: rank(Y) < J (use the S:136 completion)")
    U = (Y @ V) / np.sqrt(w[:J])
    for j in range(J):
        k = int(np.argmax(np.abs(U[:, j])))
        if U[k, j] < 0:
            U[:, j] = -U[:, j]
    return U, w


def eig_diag(w: np.ndarray, J: int) -> dict:
    """lambda_1, lambda_J, lambda_{J+1}, relative gap and kappa (§8(c) item 6)."""
    lJ = w[J - 1]
    lJ1 = w[J] if J < w.size else 0.0
    gap = lJ - lJ1
    return dict(l1=float(w[0]), lJ=float(lJ), lJ1=float(lJ1),
                rel_gap=float(gap / lJ) if lJ != 0 else 0.0,
                kappa=float(w[0] / gap) if gap > 0 else float("inf"))


def hooi_sweep(T: SparseTensor, U, core, diag=None):
    """One pass of Fig. 4's main loop body: for n = 1..N in order,
    Z <- [[X; A(1)T..I_n..A(N)T]], A(n) <- J_n leading eigenvectors of
    Z_(n) Z_(n)^T.  Gauss-Seidel: later modes use the freshly updated factors.
    Returns (U_new, Y_last) where Y_last = Z_(N) of the final mode."""
    U = [np.asarray(u, dtype=np.float64) for u in U]
    Y = None
    for n in range(T.N):
        Y = ttm_chain_unfold(T, U, n)
        S = Y @ Y.T
        U[n], w = leading_eigenvectors(S, core[n])
        if diag is not None:
            diag.append(dict(mode=n, **eig_diag(w, core[n])))
    return U, Y


def hooi_sweep_large(T: SparseTensor, U, core, diag=None):
    """:func:`hooi_sweep` for tensors whose dense intermediates do not fit: the
    projection is :func:`ttm_chain_unfold_slices` (order 3) and the factor comes
    from the smaller Gram (Y Y^T when I_n <= prod_{m != n} J_m, else Y^T Y via
    :func:`leading_left_vectors_gram_t`; reading A10: the same U_n).  Returns
    (U_new, Y_last) like hooi_sweep."""
    U = [np.asarray(u, dtype=np.float64) for u in U]
    Y = None
    for n in range(T.N):
        Y = ttm_chain_unfold_slices(T, U, n)
        if Y.shape[0] <= Y.shape[1]:
            U[n], w = leading_eigenvectors(Y @ Y.T, core[n])
        else:
            U[n], w = leading_left_vectors_gram_t(Y, core[n])
        if diag is not None:
            diag.append(dict(mode=n, **eig_diag(w, core[n])))
    return U, Y


def core_from_last_projection(U, Y_last) -> np.ndarray:
    """G from Y_(N) = (X x_{m < N} U_m^T)_(N): G_(N) = U_N^T Y_(N) (Eq. 1 for the
    last mode, Fig. 4 last step), folded to J_1 x ... x J_N (mode-1 fastest)."""
    N = len(U)
    GN = np.asarray(U[N - 1], dtype=np.float64).T @ Y_last
    dims = [u.shape[1] for u in U]
    return fold(GN, N - 1, dims)


def run_hooi_large(T: SparseTensor, U0, core_dims, sweeps: int, diag=None, log=None):
    """Fixed-sweep HOOI (Fig. 4) with :func:`hooi_sweep_large`; the core of each
    sweep comes from that sweep's last projection.  `log(msg)` (optional)
    reports progress.  Returns dict(U, G, fits, fit)."""
    U = [np.asarray(u, dtype=np.float64) for u in U0]
    nx2 = T.norm2()
    fits, G = [], None
    for t in range(sweeps):
        U, Y = hooi_sweep_large(T, U, core_dims, diag)
        G = core_from_last_projection(U, Y)
        fits.append(fit_from_core(nx2, G))
        if log:
            log(f"sweep {t + 1}: fit {fits[-1]:.10f}")
    return dict(U=U, G=G, fits=fits, fit=fits[-1])


# ---------------------------------------------------------------------------
# Multislice Projection (Fig. 7, Fig. 8, Appendix)
# ---------------------------------------------------------------------------


def mp_term_unfold(T: SparseTensor, Um: np.ndarray, n: int, m: int) -> np.ndarray:
    """W = (X x_m U_m^T)_(n): I_n x (J_m * prod_{k not in {n,m}} I_k), Kolda order.

    Its column block for one slice s (all modes other than n, m fixed) is
    P_s = X_s U_m, where X_s is the I_n x I_m slice (orientation as in Fig. 7:
    X_{::i} B for n=1, m=2)."""
    rest = [k for k in range(T.N) if k != m]
    Z = T.matrix(rest, m) @ np.asarray(Um, dtype=np.float64)
    Z = Z.reshape([T.dims[k] for k in rest] + [Um.shape[1]], order="F")
    Z = np.moveaxis(Z, -1, m)
    return unfold(Z, n)


def mp_gram(T: SparseTensor, U, n: int) -> np.ndarray:
    """M_n = sum_{m != n} sum_{slices s fixing all modes not in {n,m}} (X_s U_m)(X_s U_m)^T.

    Fig. 7 (order 3) / Fig. 8 (order 4) main-loop M_n; Appendix
    (``M1 = M1 + ((X2_slice*C)*(C'*X2_slice'))``).  Reading A1: this is a SUM of
    single-mode projections, not HOOI's chain.  The slice sum equals W W^T with
    W the column concatenation of the P_s blocks (pinned against
    :func:`mp_gram_slices`, P9)."""
    M = np.zeros((T.dims[n], T.dims[n]))
    for m in range(T.N):
        if m == n:
            continue
        W = mp_term_unfold(T, U[m], n, m)
        M += W @ W.T
    return M


def mp_gram_slices(T: SparseTensor, U, n: int) -> np.ndarray:
    """Literal slice loop of Figs. 7/8 (small inputs only): for each m != n and
    each slice s fixing the modes not in {n, m}, M_n += X_s U_m U_m^T X_s^T."""
    M = np.zeros((T.dims[n], T.dims[n]))
    for m in range(T.N):
        if m == n:
            continue
        Um = np.asarray(U[m], dtype=np.float64)
        fixed = [k for k in range(T.N) if k not in (n, m)]
        key = np.zeros_like(T.vals, dtype=np.int64)
        for k in fixed:
            key = key * T.dims[k] + T.idx[k]
        for s in np.unique(key):
            sel = key == s
            Xs = sp.csr_matrix((T.vals[sel], (T.idx[n][sel], T.idx[m][sel])),
                               shape=(T.dims[n], T.dims[m]))
            P = Xs @ Um
            M += P @ P.T
    return M


def mp_gram_rows(T: SparseTensor, U, n: int, rows, chunk: int = 2_000_000) -> np.ndarray:
    """Rows `rows` of M_n (Fig. 7/8, Appendix) without forming M_n or W:
    M_n[i, :] = sum_{m != n} sum_{slices s} P_s[i, :] P_s^T with P_s = X_s U_m (Eq. 1),
    the slices s fixing the third mode o.  The slices are visited in chunks of at most
    `chunk` nonzeros so that memory stays bounded (BASELINE config 5: d = 50000, 2e8
    nonzeros).  Order 3."""
    if T.N != 3:
        raise ValueError("mp_gram_rows: order 3 only")
    rows = np.asarray(rows, dtype=np.int64)
    out = np.zeros((rows.size, T.dims[n]))
    for m in range(3):
        if m == n:
            continue
        o = 3 - n - m
        Um = np.asarray(U[m], dtype=np.float64)
        order = np.argsort(T.idx[o], kind="stable")
        so_all = T.idx[o][order]
        bounds = np.searchsorted(so_all, np.arange(T.dims[o] + 1))  # nonzeros of slice s
        s0 = 0
        while s0 < T.dims[o]:
            s1 = max(s0 + 1, int(np.searchsorted(bounds, bounds[s0] + chunk, side="right")) - 1)
            s1 = min(s1, T.dims[o])
            sel = order[bounds[s0]:bounds[s1]]
            if sel.size:
                so, sn, sm = T.idx[o][sel], T.idx[n][sel], T.idx[m][sel]
                key = (so - s0) * T.dims[n] + sn
                uk, inv = np.unique(key, return_inverse=True)    # fibers (s, i')
                Xs = sp.csr_matrix((T.vals[sel], (inv, sm)), shape=(uk.size, T.dims[m]))
                P = Xs @ Um                                      # row (s, i') of P_s
                ks, ki = uk // T.dims[n], uk % T.dims[n]
                for k, i in enumerate(rows):
                    mine = np.flatnonzero(ki == i)               # P_s[i] of the chunk's slices
                    if mine.size == 0:
                        continue
                    Pi = np.zeros((s1 - s0, Um.shape[1]))
                    Pi[ks[mine]] = P[mine]
                    np.add.at(out[k], ki, np.einsum("fj,fj->f", P, Pi[ks]))
            s0 = s1
    return out


def mp_sweep(T: SparseTensor, U, core, diag=None):
    """One pass of Fig. 7/8's main loop: for n = 1..N, M_n as above with the
    freshest factors (Appendix: M2 uses the new A), then A(n) <- J_n leading
    eigenvectors of M_n (reading A2: of M_n itself)."""
    U = [np.asarray(u, dtype=np.float64) for u in U]
    for n in range(T.N):
        M = mp_gram(T, U, n)
        U[n], w = leading_eigenvectors(M, core[n])
        if diag is not None:
            diag.append(dict(mode=n, **eig_diag(w, core[n])))
    return U


# ---------------------------------------------------------------------------
# Slice Projection (Figs. 5-6; Wang & Ahuja).  Mode n is updated from
# ONE other factor, the previous mode's (cyclically: mode 1 from the last):
#   order 3: M13 = sum_{i in mode 2} X_{:i:} C C^T X_{:i:}^T  -> A   (n=1, m=3)
#            M21 = sum_{i in mode 3} X_{::i}^T A A^T X_{::i}  -> B   (n=2, m=1)
#            M32 = sum_{i in mode 1} X_{i::}^T B B^T X_{i::}  -> C   (n=3, m=2)
#   order 4: the same with slices fixing the two modes not in {n, m} (Fig. 6).
# Each M is one term of MP's M_n (the slices fix every mode not in {n, m}).
# ---------------------------------------------------------------------------


def sp_gram(T: SparseTensor, U, n: int) -> np.ndarray:
    """SP's M for mode n: sum over slices s fixing the modes not in {n, m},
    m = n - 1 (cyclic), of (X_s U_m)(X_s U_m)^T (Figs. 5-6)."""
    m = (n - 1) % T.N
    W = mp_term_unfold(T, np.asarray(U[m], dtype=np.float64), n, m)
    return W @ W.T


def sp_sweep(T: SparseTensor, U, core, diag=None):
    """One pass of Fig. 5/6's main loop: A(n) <- J_n leading eigenvectors of
    M (reading A2: of M itself, not M M^T), freshest factors."""
    U = [np.asarray(u, dtype=np.float64) for u in U]
    for n in range(T.N):
        U[n], w = leading_eigenvectors(sp_gram(T, U, n), core[n])
        if diag is not None:
            diag.append(dict(mode=n, **eig_diag(w, core[n])))
    return U


def run_sp(T: SparseTensor, U0, core_dims, sweeps: int):
    """Fixed-sweep SP from given factors (only the last one is used first)."""
    U = [np.asarray(u, dtype=np.float64) for u in U0]
    nx2 = T.norm2()
    fits, gn = [], []
    for _ in range(sweeps):
        U = sp_sweep(T, U, core_dims)
        G = core(T, U)
        fits.append(fit_from_core(nx2, G))
        gn.append(float(np.linalg.norm(G)))
    return dict(U=U, fits=fits, gnorms=gn)


def run_sp_converged(T: SparseTensor, core_dims, C0, tol=1e-4, maxit=50):
    """The paper's SP: random-uniform last factor C0, main loop until
    Delta_G(t) = 1 - ||G^(t-1)||_F / ||G^(t)||_F < tol or maxit (Eq. 11,
    P:874-886); ||G^(0)|| = 0, so the first sweep never stops."""
    U = [np.zeros((d, J)) for d, J in zip(T.dims, core_dims)]
    U[-1] = np.asarray(C0, dtype=np.float64)
    nx2 = T.norm2()
    gprev, it, G = 0.0, 0, None
    for it in range(1, maxit + 1):
        U = sp_sweep(T, U, core_dims)
        G = core(T, U)
        g = float(np.linalg.norm(G))
        if 1.0 - gprev / g < tol:
            break
        gprev = g
    return dict(U=U, fit=fit_from_core(nx2, G), iters=it)


# ---------------------------------------------------------------------------
# Core and fit (Fig. 4 last step P:629-631, Appendix, Eq. 9)
# ---------------------------------------------------------------------------


def core(T: SparseTensor, U) -> np.ndarray:
    """G = [[X; A(1)T, ..., A(N)T]] (Figs. 1-8 final step): dense J_1 x..x J_N."""
    Z = ttm_chain(T, U, T.N - 1)
    return ttm(Z, np.asarray(U[T.N - 1], dtype=np.float64).T, T.N - 1)


def fit_from_core(normX2: float, G: np.ndarray) -> float:
    """Eq. 9 via ||X - Xhat||^2 = ||X||^2 - ||G||^2 for orthonormal factors and
    G = [[X; U^T]] (reading A7/A8: (1 - fit)^2 = 1 - ||G||^2/||X||^2)."""
    g2 = float(np.dot(G.ravel(), G.ravel()))
    return 1.0 - np.sqrt(max(0.0, normX2 - g2)) / np.sqrt(normX2)


def fit_residual(T: SparseTensor, G: np.ndarray, U) -> float:
    """Eq. 9 by the dense residual (Appendix); small inputs only."""
    X = T.to_dense()
    return fit_dense(X, tucker_operator(G, [np.asarray(u, dtype=np.float64) for u in U]))


# ---------------------------------------------------------------------------
# Initialisations (NEXT 1) and drivers
# ---------------------------------------------------------------------------


def hosvd_factor(T: SparseTensor, n: int, J: int) -> np.ndarray:
    """A(n) <- J_n leading eigenvectors of X_(n) X_(n)^T (Fig. 2)."""
    others = [m for m in range(T.N) if m != n]
    Xn = T.matrix(others, n).T.tocsr()  # I_n x prod(others)
    S = (Xn @ Xn.T).toarray()
    return leading_eigenvectors(S, J)[0]


def pseudo_hosvd_gram(T: SparseTensor, n: int) -> np.ndarray:
    """MP's initial M_n (Fig. 7, Fig. 8):
    sum over the other modes m of sum_s X_s X_s^T for slices fixing modes not
    in {n, m}; each term equals X_(n) X_(n)^T (pin P6)."""
    M = np.zeros((T.dims[n], T.dims[n]))
    for m in range(T.N):
        if m == n:
            continue
        fixed = [k for k in range(T.N) if k not in (n, m)]
        # rows: i_n ; cols: (i_m, fixed...) -- the concatenation of the X_s blocks
        Xn = T.matrix([m] + fixed, n).T.tocsr()
        M += (Xn @ Xn.T).toarray()
    return M


def run_hooi(T: SparseTensor, U0, core_dims, sweeps: int, diag=None):
    """Fixed-sweep HOOI from given factors (reading A5/A6); U0[0] is unused
    (Fig. 3 caption P:598-602).  Returns dict(U, G, fits)."""
    U = [np.asarray(u, dtype=np.float64) for u in U0]
    nx2 = T.norm2()
    fits = []
    for _ in range(sweeps):
        U, _Y = hooi_sweep(T, U, core_dims, diag)
        fits.append(fit_from_core(nx2, core(T, U)))
    G = core(T, U)
    return dict(U=U, G=G, fits=fits, fit=fit_from_core(nx2, G))


def run_mp(T: SparseTensor, U0, core_dims, sweeps: int, diag=None):
    """Fixed-sweep MP from given factors; U0[0] is unused (Appendix
    uses B, C only to form M1)."""
    U = [np.asarray(u, dtype=np.float64) for u in U0]
    nx2 = T.norm2()
    fits = []
    for _ in range(sweeps):
        U = mp_sweep(T, U, core_dims, diag)
        fits.append(fit_from_core(nx2, core(T, U)))
    G = core(T, U)
    return dict(U=U, G=G, fits=fits, fit=fit_from_core(nx2, G))


def run_hooi_converged(T: SparseTensor, core_dims, tol=1e-4, maxit=50):
    """The paper's HOOI: HO-SVD init of modes 2..N (Fig. 4), then
    sweeps until Delta_fit < 1e-4 or 50 iterations (Eq. 10)."""
    U = [None] + [hosvd_factor(T, n, core_dims[n]) for n in range(1, T.N)]
    U[0] = np.zeros((T.dims[0], core_dims[0]))
    nx2 = T.norm2()
    old, fit, it = 0.0, 0.0, 0
    for it in range(1, maxit + 1):
        U, _ = hooi_sweep(T, U, core_dims)
        fit = fit_from_core(nx2, core(T, U))
        if fit - old < tol:
            break
        old = fit
    return dict(U=U, fit=fit, iters=it)


def run_mp_converged(T: SparseTensor, core_dims, tol=1e-4, maxit=50):
    """The paper's MP: pseudo HO-SVD init of modes 2..N (Fig. 7/8), then the
    main loop until (fit - old_fit) < 1e-4 or 50 loops (Appendix)."""
    U = [np.zeros((T.dims[0], core_dims[0]))] + [
        leading_eigenvectors(pseudo_hosvd_gram(T, n), core_dims[n])[0] for n in range(1, T.N)]
    nx2 = T.norm2()
    old, fit, it = 0.0, 0.0, 0
    for it in range(1, maxit + 1):
        U = mp_sweep(T, U, core_dims)
        fit = fit_from_core(nx2, core(T, U))
        if fit - old < tol:
            break
        old = fit
    return dict(U=U, fit=fit, iters=it)


def run_hosvd(T: SparseTensor, core_dims):
    """HO-SVD (Fig. 2): every factor from X alone, then the core and fit."""
    U = [hosvd_factor(T, n, core_dims[n]) for n in range(T.N)]
    return dict(U=U, fit=fit_from_core(T.norm2(), core(T, U)))


# ---------------------------------------------------------------------------
# Parity metrics (north star tolerances)
# ---------------------------------------------------------------------------


def projector_distance(U: np.ndarray, V: np.ndarray) -> float:
    """||U U^T - V V^T||_F (sign- and rotation-invariant) for orthonormal U, V,
    computed without the I x I projectors and without cancellation:
    ||U U^T - V V^T||^2 = J_u + J_v - 2||U^T V||^2 = ||U - V V^T U||^2 + ||V - U U^T V||^2."""
    U = np.asarray(U, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    a = U - V @ (V.T @ U)
    b = V - U @ (U.T @ V)
    return float(np.sqrt(np.sum(a * a) + np.sum(b * b)))


def rel_frobenius(A: np.ndarray, B: np.ndarray) -> float:
    B = np.asarray(B, dtype=np.float64)
    return float(np.linalg.norm(np.asarray(A, dtype=np.float64) - B) / np.linalg.norm(B))
