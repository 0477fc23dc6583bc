"""GPU parity: the CUDA path (through the C-ABI) vs the fp64 oracle.

Tolerances (BASELINE.json north star):
  Y_(n)          <= 1e-4 relative Frobenius (expect ~1e-6, fp32 storage)
  Gram / M_n     <= 1e-5 relative Frobenius (3xTF32 + fp64 accumulation)
  factors        <= 1e-4 projector distance ||U U^T - U_o U_o^T||_F
  fit            <= 1e-5 absolute
  core G         <= 1e-4 relative after Procrustes alignment (reading A3)
"""
import numpy as np
import pytest

from oracle import tucker_oracle as O
from synth import make_config, random_orthonormal, uniform_distinct_coo

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi():
    import __graft_entry__
    __graft_entry__.build()
    from paper_0711_2023_b200 import capi as c
    return c


def case(dims, nnz, core, seed=7, fseed=8):
    rng = np.random.default_rng(seed)
    idx, vals = uniform_distinct_coo(dims, nnz, rng)
    frng = np.random.default_rng(fseed)
    U0 = [random_orthonormal(I, J, frng) for I, J in zip(dims, core)]
    return idx, vals, U0


def align_core(G, U, Go, Uo):
    """Procrustes-align G to the oracle's bases: G x_n R_n^T with R_n = polar(U_n^T U_o,n)."""
    Ga = np.asarray(G, dtype=np.float64)
    for n in range(len(U)):
        M = np.asarray(U[n], dtype=np.float64).T @ Uo[n]
        a, _, bt = np.linalg.svd(M)
        R = a @ bt
        Ga = O.ttm(Ga, R.T, n)
    return Ga


SHAPES = [
    ((100, 100, 100), 10_000, (10, 10, 10)),       # config 1
    ((100, 110, 120), 13_200, (10, 11, 12)),       # non-cubic (Appendix `test`)
    ((37, 300, 53), 9_000, (5, 16, 7)),            # ragged, one mode much longer (Y^T Y route)
    ((20, 22, 18, 16), 12_000, (4, 5, 3, 6)),      # order 4
]


@pytest.mark.parametrize("kernel", ["auto", "tc", "simt"])
@pytest.mark.parametrize("dims,nnz,core", SHAPES)
def test_ttmc_parity(capi, monkeypatch, dims, nnz, core, kernel):
    """Both order-3 Kronecker kernels (tcgen05 3xTF32 and SIMT fp32) and the
    default dispatch agree with the oracle's Y_(n)."""
    if kernel != "auto":
        if len(dims) != 3:
            pytest.skip("order 4 has one kernel")
        monkeypatch.setenv("TUCKER_TTMC", kernel)
    idx, vals, U0 = case(dims, nnz, core)
    T = O.SparseTensor(dims, idx, vals)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        for n in range(len(dims)):
            Y = t.debug_ttmc(n)
            Yo = O.ttm_chain_unfold(T, U0, n)
            assert O.rel_frobenius(Y, Yo) < 1e-4


@pytest.mark.parametrize("kernel", ["tc", "simt"])
@pytest.mark.parametrize("lmax,cmax", [(None, None), ("7", "3000"), ("64", "20000")])
def test_ttmc_parity_skewed(capi, monkeypatch, lmax, cmax, kernel):
    """Zipf-skewed tensor (config 5's index law at oracle size): long fibers and
    heavy head slices.  With the env hooks the SpTTMc work plan cuts fibers
    into virtual fibers of <= lmax nonzeros and slices into units of <= cmax
    work; Y must not depend on the cut (Eq. 1 is linear in t_f)."""
    from synth.generators import zipf_coo
    dims, nnz, core = (60, 70, 900), 30_000, (6, 5, 4)
    idx, vals = zipf_coo(dims, nnz, np.random.default_rng(11), batch=1 << 14)
    frng = np.random.default_rng(12)
    U0 = [random_orthonormal(I, J, frng) for I, J in zip(dims, core)]
    monkeypatch.setenv("TUCKER_TTMC", kernel)
    if lmax:
        monkeypatch.setenv("TUCKER_TTMC_LMAX", lmax)
        monkeypatch.setenv("TUCKER_TTMC_CMAX", cmax)
    T = O.SparseTensor(dims, idx, vals)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        st = t.csf_stats()
        if lmax:
            assert all(vf > f and u > 0 for f, _, vf, u in st), st
        for n in range(len(dims)):
            Y = t.debug_ttmc(n)
            Yo = O.ttm_chain_unfold(T, U0, n)
            assert O.rel_frobenius(Y, Yo) < 1e-4
        fits = t.hooi_sweep(2)
    # the whole sweep on the split path agrees with the oracle
    ref = O.run_hooi(T, U0, core, 2)
    assert np.max(np.abs(np.asarray(fits) - np.asarray(ref["fits"]))) < 1e-5


@pytest.mark.parametrize("cs,gmem", [(None, None), ("1", None), ("2", "1"), ("8", None), ("4", "1")])
def test_ttmc_parity_order4_clusters(capi, monkeypatch, cs, gmem):
    """Order 4 (k_spttmc4w): every slice split over a thread-block cluster of
    1/2/4/8 CTAs whose partial rows are summed through distributed shared memory,
    with the factor tables in shared memory or read from global memory; Y and a
    HOOI sweep agree with the oracle, and the result is bit-identical across
    cluster sizes' repeated runs."""
    dims, nnz, core = (20, 22, 18, 16), 12_000, (4, 5, 3, 6)
    idx, vals, U0 = case(dims, nnz, core)
    if cs:
        monkeypatch.setenv("TUCKER_TTMC4_CS", cs)
    if gmem:
        monkeypatch.setenv("TUCKER_TTMC4_GMEM", gmem)
    T = O.SparseTensor(dims, idx, vals)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        for n in range(4):
            Y = t.debug_ttmc(n)
            assert O.rel_frobenius(Y, O.ttm_chain_unfold(T, U0, n)) < 1e-4
            np.testing.assert_array_equal(Y, t.debug_ttmc(n))
        fits = t.hooi_sweep(2)
    ref = O.run_hooi(T, U0, core, 2)
    assert np.max(np.abs(np.asarray(fits) - np.asarray(ref["fits"]))) < 1e-5


@pytest.mark.parametrize("dims,nnz,core", [((9, 40, 33, 7), 6_000, (3, 8, 12, 2)),
                                            ((30, 6, 5, 50), 4_000, (7, 2, 5, 9)),
                                            ((12, 13, 14, 15), 20_000, (2, 3, 5, 7))])
def test_ttmc_parity_order4_shapes(capi, dims, nnz, core):
    """Ragged order-4 shapes: core sizes that are not multiples of 4 (padded
    factor rows), empty slices and nodes, and different leaf / mid choices."""
    idx, vals, U0 = case(dims, nnz, core)
    T = O.SparseTensor(dims, idx, vals)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        for n in range(4):
            assert O.rel_frobenius(t.debug_ttmc(n), O.ttm_chain_unfold(T, U0, n)) < 1e-4


@pytest.mark.parametrize("dims,nnz,core", [((9, 40, 33, 7), 6_000, (3, 8, 12, 2)),
                                            ((30, 6, 5, 50), 4_000, (7, 2, 5, 9)),
                                            ((12, 13, 14, 15), 20_000, (2, 3, 5, 7)),
                                            ((20, 22, 18, 16), 12_000, (4, 5, 3, 6)),
                                            ((40, 200, 30, 20), 48_000, (5, 6, 20, 8)),
                                            ((7, 300, 37, 21), 60_000, (3, 21, 9, 13))])
@pytest.mark.parametrize("kern", ["g", "t", "s"])
def test_ttmc_parity_order4_gemm(capi, monkeypatch, dims, nnz, core, kern):
    """Order-4 GEMM-form SpTTMc (k_spttmc4g on the FMA pipes, k_spttmc4t with level 2
    on tcgen05 in 3xTF32; forced with TUCKER_TTMC4=g / t even where the dispatch
    would pick k_spttmc4w): the dense batch layout (partial last
    batches, mid1 ranges that are not multiples of the 16-index chunk, empty
    slices and nodes), several batches per slice and per CTA (runs summed in
    batch order) and ragged core sizes; Y equals the oracle's and the old
    kernel's, repeated runs are bit-identical, and a HOOI sweep matches."""
    idx, vals, U0 = case(dims, nnz, core)
    T = O.SparseTensor(dims, idx, vals)
    monkeypatch.setenv("TUCKER_TTMC4", kern)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        Yg = [t.debug_ttmc(n) for n in range(4)]
        for n in range(4):
            assert O.rel_frobenius(Yg[n], O.ttm_chain_unfold(T, U0, n)) < 1e-4
            np.testing.assert_array_equal(Yg[n], t.debug_ttmc(n))
        fits = t.hooi_sweep(1)
    monkeypatch.setenv("TUCKER_TTMC4", "w")
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        for n in range(4):
            assert O.rel_frobenius(Yg[n], t.debug_ttmc(n)) < 1e-5
    ref = O.run_hooi(T, U0, core, 1)
    assert np.max(np.abs(np.asarray(fits) - np.asarray(ref["fits"]))) < 1e-5


@pytest.mark.parametrize("dims,nnz,core", SHAPES)
def test_gram_parity(capi, dims, nnz, core):
    idx, vals, U0 = case(dims, nnz, core)
    T = O.SparseTensor(dims, idx, vals)
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        for n in range(len(dims)):
            S = t.debug_gram(0, n)
            Yo = O.ttm_chain_unfold(T, U0, n)
            assert O.rel_frobenius(S, Yo @ Yo.T) < 1e-5
            M = t.debug_gram(1, n)
            assert O.rel_frobenius(M, O.mp_gram(T, U0, n)) < 1e-5


@pytest.mark.parametrize("d,J,gap", [(100, 10, 1e-2), (300, 50, 1e-3), (1000, 50, 3e-4), (250, 100, 1e-2)])
def test_eig_parity(capi, d, J, gap):
    rng = np.random.default_rng(d + J)
    Q = np.linalg.qr(rng.standard_normal((d, d)))[0]
    # a dominant "mean" eigenvalue, a flat bulk and a small J/J+1 gap
    w = np.sort(rng.uniform(0.1, 1.0, d))[::-1].copy()
    w[0] = 60.0
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
    np.testing.assert_allclose(ev, wo[:J], rtol=1e-10)
    # sign canonical and ordered
    for j in range(J):
        k = int(np.argmax(np.abs(U[:, j])))
        assert U[k, j] > 0


def run_both(capi, dims, idx, vals, U0, core, sweeps):
    T = O.SparseTensor(dims, idx, vals)
    out = {}
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        fh = t.hooi_sweep(sweeps)
        G, U, fit = t.core_and_fit()
        out["hooi"] = (fh, G, U, fit)
        t.set_factors(U0)
        fm = t.mp_sweep(sweeps)
        Gm, Um, fitm = t.core_and_fit()
        out["mp"] = (fm, Gm, Um, fitm)
    dh, dm = [], []
    ref = {"hooi": O.run_hooi(T, U0, core, sweeps, diag=dh), "mp": O.run_mp(T, U0, core, sweeps, diag=dm)}
    # the conditioning of every factor update the parity rests on
    N = len(dims)
    for algo, dg in (("hooi", dh), ("mp", dm)):
        for i, d in enumerate(dg):
            print(f"kappa {algo} sweep {i // N} mode {d['mode'] + 1}: lambda_1 {d['l1']:.6g} "
                  f"lambda_J {d['lJ']:.6g} lambda_J+1 {d['lJ1']:.6g} rel_gap {d['rel_gap']:.3g} "
                  f"kappa {d['kappa']:.4g}")
    ref["hooi"]["diag"], ref["mp"]["diag"] = dh, dm
    return out, ref


@pytest.mark.parametrize("dims,nnz,core", SHAPES)
def test_end_to_end_parity(capi, dims, nnz, core):
    idx, vals, U0 = case(dims, nnz, core)
    out, ref = run_both(capi, dims, idx, vals, U0, core, 3)
    for algo in ("hooi", "mp"):
        fits, G, U, fit = out[algo]
        r = ref[algo]
        for n in range(len(dims)):
            assert O.projector_distance(U[n], r["U"][n]) < 1e-4, (algo, n)
            assert np.abs(U[n].astype(np.float64).T @ U[n] - np.eye(core[n])).max() < 1e-5
        assert abs(fit - r["fit"]) < 1e-5
        np.testing.assert_allclose(fits, r["fits"], atol=1e-5)
        Ga = align_core(G, U, r["G"], r["U"])
        assert O.rel_frobenius(Ga, r["G"]) < 1e-4


def test_config1_full(capi):
    c = make_config(1)
    out, ref = run_both(capi, c["dims"], c["idx"], c["vals"], c["U0"], c["core"], c["sweeps"])
    for algo in ("hooi", "mp"):
        _, _, U, fit = out[algo]
        for n in range(3):
            assert O.projector_distance(U[n], ref[algo]["U"][n]) < 1e-4
        assert abs(fit - ref[algo]["fit"]) < 1e-5


@pytest.mark.parametrize("k", [2, 3, 4])
def test_config_full(capi, k, record_property):
    """BASELINE.json configs[k-1] at full size from the seeded U0 with their full
    5 HOOI + 5 MP sweeps: config 2 (1000^3, 1e6 nnz, core 50^3), config 3 (2000^3,
    8e6 nnz, unbalanced core 100x25x10) and config 4 (order 4, 200^4, 1.6e7 nnz, the
    bench's workload).  Factors (projector distance), fits per sweep and the core
    (after Procrustes alignment) vs the oracle; kappa of every update is printed and
    recorded."""
    c = make_config(k)
    sw = c["sweeps"]
    out, ref = run_both(capi, c["dims"], c["idx"], c["vals"], c["U0"], c["core"], sw)
    record_property("kappa", {a: [round(d["kappa"], 3) for d in ref[a]["diag"]] for a in ("hooi", "mp")})
    for algo in ("hooi", "mp"):
        fits, G, U, fit = out[algo]
        r = ref[algo]
        for n in range(len(c["dims"])):
            d = O.projector_distance(U[n], r["U"][n])
            assert d < 1e-4, (algo, n, d)
        assert abs(fit - r["fit"]) < 1e-5
        np.testing.assert_allclose(fits, r["fits"], atol=1e-5)
        Ga = align_core(G, U, r["G"], r["U"])
        assert O.rel_frobenius(Ga, r["G"]) < 1e-4


def test_edge_cases(capi):
    dims, core = (30, 40, 25), (3, 4, 2)
    idx, vals, U0 = case(dims, 600, core)
    # duplicate coordinate
    idx_d = [np.concatenate([a, a[:1]]) for a in idx]
    with pytest.raises(capi.TuckerError) as e:
        capi.Tucker(dims, core, idx_d, np.concatenate([vals, vals[:1]]), U0)
    assert e.value.code == 3
    # out of range
    idx_o = [a.copy() for a in idx]
    idx_o[2][5] = dims[2]
    with pytest.raises(capi.TuckerError) as e:
        capi.Tucker(dims, core, idx_o, vals, U0)
    assert e.value.code == 2
    # non-finite value
    v = vals.copy()
    v[3] = np.nan
    with pytest.raises(capi.TuckerError) as e:
        capi.Tucker(dims, core, idx, v, U0)
    assert e.value.code == 4
    # all-zero tensor
    with pytest.raises(capi.TuckerError) as e:
        capi.Tucker(dims, core, idx, np.zeros_like(vals), U0)
    assert e.value.code == 4
    # explicit zeros are dropped; empty slices (mode-1 indices >= 20 unused) are fine
    v = vals.copy()
    v[::7] = 0
    idx_e = [a.copy() for a in idx]
    idx_e[0] = idx_e[0] % 20
    keep = np.unique(np.stack(idx_e), axis=1, return_index=True)[1]
    idx_e = [a[np.sort(keep)] for a in idx_e]
    v = v[np.sort(keep)]
    out, ref = run_both(capi, dims, idx_e, v, U0, core, 2)
    for algo in ("hooi", "mp"):
        _, _, U, fit = out[algo]
        assert abs(fit - ref[algo]["fit"]) < 1e-5
        for n in range(3):
            assert O.projector_distance(U[n], ref[algo]["U"][n]) < 1e-4


def test_determinism(capi):
    dims, core = (60, 50, 40), (6, 5, 4)
    idx, vals, U0 = case(dims, 5000, core)
    res = []
    for _ in range(2):
        with capi.Tucker(dims, core, idx, vals, U0) as t:
            t.hooi_sweep(2)
            G, U, fit = t.core_and_fit()
            res.append((G, U, fit))
    assert res[0][2] == res[1][2]
    np.testing.assert_array_equal(res[0][0], res[1][0])
    for a, b in zip(res[0][1], res[1][1]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("algo", ["hooi", "mp"])
def test_convergence_driver(capi, algo):
    """hooi_run / mp_run (Eq. 10 stop rule, NEXT 2): the per-sweep fits match the
    oracle's sweeps from the same U0, and the loop stops at the first sweep
    whose Delta_fit < tol (tol chosen away from the measured increments)."""
    dims, nnz, core = (100, 100, 100), 10_000, (10, 10, 10)
    idx, vals, U0 = case(dims, nnz, core)
    T = O.SparseTensor(dims, idx, vals)
    ref = (O.run_hooi if algo == "hooi" else O.run_mp)(T, U0, core, 12)["fits"]
    inc = np.diff(np.concatenate([[0.0], ref]))
    # a tolerance below every earlier increment and above the stopping one
    k = next(i for i in range(2, len(inc)) if inc[i] < 0.5 * inc[:i].min())
    tol = float(np.sqrt(inc[k] * inc[:k].min()))
    with capi.Tucker(dims, core, idx, vals, U0) as t:
        fits = getattr(t, algo + "_run")(max_sweeps=50, tol=tol)
    assert len(fits) == k + 1
    assert np.max(np.abs(fits - ref[: k + 1])) < 1e-5


@pytest.mark.parametrize("dims,nnz,core", [((100, 110, 120), 13_200, (10, 11, 12)),
                                            ((20, 22, 18, 16), 12_000, (4, 5, 3, 6)),
                                            ((200, 200, 200, 200), 400_000, (20, 20, 20, 20))])
def test_mp_overlap(capi, monkeypatch, dims, nnz, core):
    """MP sweep with the next mode's early terms (W columns and their Gram into S2) built on a
    second stream while the eigensolve runs, the late term added on the main stream: the same
    sums in another fp64 order -- fits and factors agree with the serial sweep to rounding, and
    both with the oracle."""
    idx, vals, U0 = case(dims, nnz, core)
    out = {}
    for ov in ("0", "1"):
        monkeypatch.setenv("TUCKER_MP_OVERLAP", ov)
        with capi.Tucker(dims, core, idx, vals, U0) as t:
            f = t.mp_sweep(3)
            G, U, fit = t.core_and_fit()
        out[ov] = (np.asarray(f), U, fit)
    f0, U0g, _ = out["0"]
    f1, U1g, _ = out["1"]
    assert np.max(np.abs(f0 - f1)) < 1e-9
    for a, b in zip(U0g, U1g):
        assert O.projector_distance(a, b) < 1e-4  # fp32 factors of an ill-conditioned sum (kappa ~1e3)
    if nnz <= 20_000:
        T = O.SparseTensor(dims, idx, vals)
        ref = O.run_mp(T, U0, core, 3)
        assert np.max(np.abs(f1 - np.asarray(ref["fits"]))) < 1e-5
