/*
 * tucker.h -- C-ABI of libtucker.so, the B200 (sm_100a) hot path shared by HOOI
 * and Multislice Projection (MP) from arxiv/paper_0711_2023.
 *
 * Citations: P:<line> = PAPER.md line.  Operation set: SURVEY.md §8(b).
 *
 * Conventions (all entry points)
 *   - order N, dims I_1..I_N, core J_1..J_N (Eq. 8): "Tucker
 *     decomposition X ~ [[G; A(1)..A(N)]]", A(n) is I_n x J_n with orthonormal
 *     columns.
 *   - Indices are 0-BASED int32 (the paper's text files are 1-based).
 *   - Nonzero values are fp32; explicit zeros are accepted and dropped.
 *   - Factor matrices are fp32, ROW-MAJOR I_n x J_n (element (i,j) at i*J_n+j).
 *   - The core G is fp32, mode-1 fastest: G(j1..jN) at j1 + J1*(j2 + J2*(...)).
 *   - Unfoldings Y_(n) use the Kolda column order (Eqs. 3-6): the
 *     remaining modes in increasing order, lower modes varying fastest.
 *   - All calls are blocking (stream-synchronised on return) and not
 *     re-entrant per handle.  Different handles may be used from different
 *     threads.
 *   - Multi-GPU: one process per GPU;
 *     every rank passes the FULL tensor and the same arguments, plus its rank,
 *     the world size and the same 128-byte ncclUniqueId (tucker_nccl_unique_id
 *     on one rank, broadcast by the caller).  hooi_sweep, mp_sweep,
 *     core_and_fit and the debug Gram/TTMc calls are then collective: every
 *     rank makes the same call sequence (the debug Gram returns this rank's
 *     partial Gram).  The library picks its own shard
 *     (HOOI: a contiguous range of mode-n slices, MP: of each term's slice
 *     index) and sums partial results with NCCL allreduces on its stream;
 *     factors, core and fit come back replicated on every rank.
 *
 * Return value: 0 (TUCKER_OK) or one of the TUCKER_E_* codes below; a
 * human-readable message for the code is tucker_strerror(code) and the last
 * detailed message of a handle is tucker_last_error(h).
 *
 * Ownership: tucker_init copies every input; the caller may free them on
 * return.  The handle owns all device memory it allocates.  Output buffers are
 * caller-owned host (or, with TUCKER_OUTPUT_ON_DEVICE, device) memory.
 */
#ifndef TUCKER_H
#define TUCKER_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TUCKER_OK 0
#define TUCKER_E_ARG 1     /* null pointer, order/dims/core/nnz/sweeps out of range          */
#define TUCKER_E_INDEX 2   /* an index outside [0, I_n)                                        */
#define TUCKER_E_DUP 3     /* duplicate coordinate                                */
#define TUCKER_E_VALUE 4   /* non-finite value, or ||X|| = 0 (fit undefined, Eq. 9)            */
#define TUCKER_E_FACTOR 5  /* initial factor not orthonormal (max|U^T U - I| > 1e-5)           */
#define TUCKER_E_CUDA 6    /* CUDA runtime error (message in tucker_last_error)                */
#define TUCKER_E_NCCL 7    /* NCCL error                                                       */
#define TUCKER_E_OOM 8     /* device allocation failed                                         */
#define TUCKER_E_STATE 9   /* call out of order (e.g. a debug query before it is available)    */
#define TUCKER_E_CONVERGE 10 /* eigensolver hit its iteration cap above tolerance (result kept) */

/* flags */
#define TUCKER_INPUT_ON_DEVICE 0x1u   /* idx/vals/U0 pointers are device pointers                */
#define TUCKER_OUTPUT_ON_DEVICE 0x2u  /* core_out/U_out/Y/S outputs are device pointers          */
#define TUCKER_HOST_COLLECTIVES 0x4u  /* world > 1 without NCCL: the sharded sweep's sums go through
                                         the callback of tucker_set_allreduce (tests; other layers)  */

typedef struct tucker_handle tucker_handle;

typedef struct {
  int device;                 /* CUDA device ordinal for this rank                             */
  int rank, world;            /* one rank per GPU, 0 <= rank < world                           */
  const void* nccl_unique_id; /* 128-byte ncclUniqueId, required when world > 1; with world == 1
                                 it runs the sharded code path over a 1-rank communicator       */
  void* stream;               /* cudaStream_t to run on (NULL = the handle's own stream)        */
  int eig_oversample;         /* p in block size k = J + p (0 = default)         */
  int eig_max_iter;           /* cap on Chebyshev-filter outer iterations (0 = default 60)      */
  double eig_tol;             /* Ritz residual tolerance relative to theta_1 (0 = default)      */
  unsigned flags;             /* TUCKER_* flags above                                           */
} tucker_opts;

/* Fill *opts with defaults (device 0, world 1, own stream). */
void tucker_default_opts(tucker_opts* opts);

/*
 * tucker_init -- load an order-N sparse tensor and the initial factors.
 *
 *   order   N in 2..8.  HOOI (Fig. 4) is defined for any N; order 2 is the
 *           matrix case.  MP and SP are defined for orders 3 and 4 only
 *           (Figs. 5-8; SURVEY reading A18): for orders 2 and 5..8 mp_sweep,
 *           sp_sweep, tucker_hosvd and the CSF queries return TUCKER_E_ARG, HOOI runs on
 *           one rank (world > 1 -> TUCKER_E_ARG) through per-mode sorted COO slices
 *           (no CSF), and the orders 3 / 4 keep the CSF kernels.
 *   dims    I_1..I_N, each >= 1 and I_n < 2^31, with prod_n I_n < 2^64 (the
 *           sort keys pack every coordinate into 64 bits; TUCKER_E_ARG otherwise).
 *   core    J_1..J_N, 1 <= J_n <= min(I_n, 240) (the eigensolvers' block k = J + p
 *           <= 256; J_n > 112 runs the host-driven solver, core sizes > 128 the
 *           tcgen05 SpTTMc in 128-column windows) and J_n <= prod_{q != n} J_q (Y_(n) has at most that
 *           rank, so no J_n-dimensional dominant subspace exists beyond it);
 *           TUCKER_E_ARG otherwise.
 *   nnz     number of COO entries (>= 1).
 *   idx     N pointers to int32[nnz], 0-based coordinates (any order).
 *   vals    fp32[nnz].
 *   U0      N pointers to fp32 I_n x J_n row-major, orthonormal columns (the
 *           north star's seeded random orthonormal factors; SURVEY reading A5).
 *           HOOI ignores U0[0] (Fig. 3 caption P:598-602); MP ignores U0[0]
 *           too (Appendix P:1818-1830 forms M1 from B, C only).
 *   opts    NULL for defaults.
 * Work: copies inputs to the device, validates them, builds the sorted
 * slice/fiber structures (CSF) for every ordering the sweeps need (the paper's
 * "sort by mode n, one slice per index" step, done in HBM), and
 * computes ||X||_F^2 in fp64.
 * Errors: E_ARG, E_INDEX, E_DUP, E_VALUE, E_FACTOR, E_OOM, E_CUDA.
 */
int tucker_init(tucker_handle** out, int order, const int64_t* dims, const int64_t* core,
                int64_t nnz, const int32_t* const* idx, const float* vals,
                const float* const* U0, const tucker_opts* opts);

/*
 * hooi_sweep -- `sweeps` passes of HOOI's main loop (Fig. 4): for
 * n = 1..N, Y_(n) = (X x_{m != n} U_m^T)_(n) (SpTTMc), S = Y Y^T or Y^T Y
 * (whichever is smaller, fp64), U_n = J_n leading eigenvectors (descending,
 * sign-canonical: largest |entry| positive).  Gauss-Seidel order.
 *   fit_per_sweep  nullable, double[sweeps]: Eq. 9 fit after each sweep.
 *   stage_ms       nullable, float[sweeps * 4]: per sweep {spttmc, gram, eig, corefit} ms.
 * Errors: E_ARG (sweeps < 1), E_CUDA, E_CONVERGE (factors still returned).
 */
int hooi_sweep(tucker_handle* h, int sweeps, double* fit_per_sweep, float* stage_ms);

/*
 * mp_sweep -- `sweeps` passes of MP's main loop (Fig. 7, Fig. 8
 * P:1040-1096, Appendix): for n = 1..N,
 *   M_n = sum_{m != n} sum_{slices s fixing the modes not in {n,m}} (X_s U_m)(X_s U_m)^T
 * (fp64, I_n x I_n), U_n = J_n leading eigenvectors of M_n (SURVEY reading A2:
 * of M_n, not M_n M_n^T).  Same output arguments as hooi_sweep
 * (stage_ms entries: {spmm, gram, eig, corefit}).  Orders 3 and 4 only (E_ARG otherwise).
 */
int mp_sweep(tucker_handle* h, int sweeps, double* fit_per_sweep, float* stage_ms);

/*
 * core_and_fit -- G = [[X; U_1^T..U_N^T]] (Figs. 1-8 final step) and
 * fit = 1 - sqrt(max(0, ||X||^2 - ||G||^2)) / ||X|| (Eq. 9 with the norm
 * identity for orthonormal factors; SURVEY readings A7/A8).
 *   core_out  nullable, fp32[prod J], mode-1 fastest.
 *   U_out     nullable, N nullable pointers to fp32 I_n x J_n row-major.
 *   fit_out   nullable.
 */
int core_and_fit(tucker_handle* h, float* core_out, float* const* U_out, double* fit_out);

/* Overwrite the handle's current factors (same layout as U0); lets a caller
 * restart HOOI/MP from the same U0 without rebuilding the CSF. */
int tucker_set_factors(tucker_handle* h, const float* const* U);

/* Release all device memory.  NULL is accepted. */
int tucker_free(tucker_handle* h);

const char* tucker_strerror(int code);
const char* tucker_last_error(const tucker_handle* h);

/* ------------------------------------------------------------------------
 * Diagnostic entry points (used by the parity tests; same kernels as the
 * sweeps, no side effect on the factors).
 * ---------------------------------------------------------------------- */

/* Y_(n) = (X x_{m != n} U_m^T)_(n) with the handle's CURRENT factors:
 * fp32 I_n x prod_{m!=n} J_m row-major, Kolda column order.  mode is 0-based. */
int tucker_debug_ttmc(tucker_handle* h, int mode, float* Y_out);

/* The fp64 Gram that the next update of `mode` would diagonalise, with the
 * current factors: algo 0 = HOOI (S = Y Y^T, I_n x I_n, always returned in this
 * orientation), algo 1 = MP (M_n, I_n x I_n).  Row-major fp64. */
int tucker_debug_gram(tucker_handle* h, int algo, int mode, double* S_out);

/* Rows `rows[0..nrows)` (0-based) of the same Gram (algo 0 HOOI, 1 MP), fp64, into
 * out (host, nrows x I_mode row-major): the Gram is formed on the device and only the
 * requested rows are copied back -- for Grams too large to return (MP at config 5:
 * 50000 x 50000).  E_ARG on bad arguments or rows out of range. */
int tucker_debug_gram_rows(tucker_handle* h, int algo, int mode, int nrows, const int64_t* rows, double* out);

/* Leading-J eigenvectors (descending, sign-canonical, fp32 row-major d x J) and
 * eigenvalues (fp64[J]) of a caller-provided symmetric fp64 d x d matrix, with
 * the library's eigensolver.  1 <= J <= min(d, 112). */
int tucker_debug_eig(tucker_handle* h, int d, int J, const double* S, float* U_out,
                     double* evals_out);

/* Unit test of the eigensolver's shared-memory k x k routines (1 <= k <= 116,
 * one CTA on the current device; no handle).  mode 0: CholQR factor of the SPD
 * matrix `in` (k x k row-major): out = M, upper triangular, with M^T in M = I
 * (`shift` is added to the equilibrated matrix as in shifted CholQR).  mode 1:
 * cyclic Jacobi with at most max_sweeps sweeps: out = V (eigenvectors in
 * columns), theta = eigenvalues in descending order, sweeps[0] = sweeps used
 * and (mode 1) sweeps[1..7] = cycle counters of thread 0 (rotation, rows, row
 * barrier, columns, column barrier, rounds, total); sweeps needs 8 entries. */
int tucker_debug_smalldense(int mode, int k, const double* in, double* out, double* theta,
                            int* sweeps, int max_sweeps, double shift);

/* Unit test of the eigensolver's fp64 tensor-core product (all SMs, no handle):
 * out = alpha S Y + gamma D with S d x d, Y, D, out d x n row-major (1 <= n <= 116;
 * D nullable). */
int tucker_debug_product(int d, int n, const double* S, const double* Y, double alpha, double gamma,
                         const double* D, double* out);

/* Timing of the same product alone: *us = microseconds per launch (mean of reps). */
int tucker_debug_product_time(int d, int n, int reps, double* us);

/* Measurement entry point: the HOOI projection of `mode` (0-based) with the
 * handle's current factors, run `reps` >= 1 times back to back on the handle's
 * stream after one untimed run; *ms_out = mean milliseconds per projection
 * (CUDA events around the repetitions: the SpTTMc kernels and the zero fill of
 * the Y buffer).  Leaves the handle's cached core invalid.  E_ARG on bad
 * arguments. */
int tucker_time_ttmc(tucker_handle* h, int mode, int reps, float* ms_out);

/* Measurement: kernel time of mp_sweep's overlapped streams (MP overlap: while mode n's
 * eigensolve runs on its own stream, a side stream builds the next mode's W terms that do not
 * involve U_n and their Gram; the main stream adds the late term m = n - 1), summed over the
 * sweeps since the last reset from CUDA events on the stream each kernel runs on.
 * ms[5] / counts[5]: [0] side SpMM (counts in terms = k_spmm_w launches), [1] side Gram (calls),
 * [2] main-stream SpMM (late term, or a whole build when nothing was prepared; terms),
 * [3] main-stream Gram (calls), [4] eigensolve + factor update (calls).  The streams overlap, so
 * the sums exceed the sweep's wall time.  The side work of a call's last mode is counted only if
 * it had finished at the sweep's end.  All zero when the overlap is off.  E_ARG on null pointers. */
int tucker_mp_overlap_times(tucker_handle* h, double* ms, int64_t* counts, int reset);

/* Sparse layout of the handle, for the CSF ordering mode n's HOOI projection
 * uses (out has 4 N entries): out[4n] = fibers, out[4n + 1] = nonzeros,
 * out[4n + 2] = virtual fibers of the SpTTMc work plan and out[4n + 3] = its
 * work units (both 0 when the tensor needs no plan: one CTA per slice). */
int tucker_csf_stats(tucker_handle* h, int64_t* out);

/* The CSF ordering each mode's HOOI projection uses (out has 8 N entries):
 * out[8n .. 8n+7] = root mode, mid0 mode, mid1 mode (-1 at order 3), leaf mode
 * (0-based), fibers (distinct root/mid coordinates), nodes (order 4: distinct
 * (root, mid0); order 3: 0), nonzeros, root slices. */
int tucker_csf_layout(tucker_handle* h, int64_t* out);

/* Kernel statistics of the handle since the last reset (for bench/roofline):
 * stats[0] = kernel launches issued by the library, [1] = eigensolver outer
 * iterations, [2] = Chebyshev matvecs, [3] = small (k x k) Jacobi sweeps,
 * [4] = Gram path (0 = by size: fp64 DMMA up to 2e10 FMA, tcgen05 3xTF32 above; 1 = fp64 DMMA for every Gram, env TUCKER_GRAM_FP64=1), [5..12] = time inside the
 * fused eigensolver kernel by phase in ns as seen by its CTA 0 (matvec, k x k
 * reductions, CholQR factor, Jacobi, row-block apply, deflation, power/Lanczos,
 * other), [13] = algorithmic fp64 flops of the eigensolver (products 2 d^2 n,
 * Grams, applies, CholQR, Jacobi rotations, deflation), [14..17] = product
 * breakdown in ns (phase A, inner barrier, phase B, leading barrier; CTA 0's
 * view).  stats has 18 entries. */
int tucker_stats(tucker_handle* h, int64_t* stats, int reset);

/* HO-SVD initialisation (NEXT 1 of SURVEY.md §8(f)): for every mode n with bit
 * n of mode_mask set, U_n <- the J_n leading eigenvectors of X_(n) X_(n)^T
 * (Fig. 2; HOOI's init of modes 2..N, Fig. 4; MP's pseudo
 * HO-SVD (N-1) X_(n) X_(n)^T has the same eigenvectors, Fig. 7), sign-
 * canonicalised, written into the handle's factors.  The sparse Gram is formed
 * from the fibers of an ordering with leaf n (pairs sorted and reduced in a
 * fixed order: deterministic).  TUCKER_E_ARG for bits >= order; TUCKER_E_OOM
 * when a mode has more than 2^31 fiber pairs; TUCKER_E_CONVERGE as the sweeps.
 * Collective when sharded (each rank a fiber range, S allreduced). */
int tucker_hosvd(tucker_handle* h, unsigned mode_mask);

/* Slice Projection (NEXT 3 of SURVEY.md §8(f); Figs. 5-6): one sweep
 * updates U_n, n = 1..N, from the single multislice term of the previous
 * mode's factor (m = n - 1, cyclic: U_1 from U_N), i.e. the J_n leading
 * eigenvectors of sum_s (X_s U_m)(X_s U_m)^T over the slices s fixing the
 * modes not in {n, m}; then the core.  fits / gnorms (nullable, length
 * sweeps): fit and ||G||_F after each sweep.  Collective when sharded. */
int sp_sweep(tucker_handle* h, int sweeps, double* fits, double* gnorms, float* stage_ms);
/* SP until Delta_G(t) = 1 - ||G^(t-1)||_F / ||G^(t)||_F < tol (Eq. 11; the
 * paper: 1e-4) or max_sweeps (50); as hooi_run otherwise. */
int sp_run(tucker_handle* h, int max_sweeps, double tol, double* fits, int* sweeps_done);
/* Replace factor n (I_n x J_n fp32 row-major, host or -- with
 * TUCKER_INPUT_ON_DEVICE -- device).  check = 1: must be orthonormal
 * (TUCKER_E_FACTOR); check = 0: any finite matrix, for SP's random-uniform
 * column-normalised initial factor. */
int tucker_set_factor(tucker_handle* h, int n, const float* U, int check);

/* The paper's stop rule (Eq. 10; MP: Appendix, NEXT 2 of
 * SURVEY.md §8(f)): sweep from the factors in the handle until
 * Delta_fit(t) = fit(t) - fit(t-1) < tol (fit(0) = 0; the paper uses 1e-4) or
 * max_sweeps sweeps (the paper: 50).  fits: per-sweep fit (length max_sweeps,
 * nullable); *sweeps_done (nullable) = sweeps run.  TUCKER_E_ARG on a null
 * handle, max_sweeps < 1 or tol < 0; TUCKER_E_CONVERGE if some eigensolve did
 * not reach its tolerance (the loop still completes).  Collective when sharded. */
int hooi_run(tucker_handle* h, int max_sweeps, double tol, double* fits, int* sweeps_done);
int mp_run(tucker_handle* h, int max_sweeps, double tol, double* fits, int* sweeps_done);

/* A fresh 128-byte ncclUniqueId in id_out (caller-owned) for tucker_opts;
 * loads NCCL (libnccl.so.2) on demand.  TUCKER_E_NCCL if it cannot. */
int tucker_nccl_unique_id(void* id_out);

/* The library's shard rule, host only (no device work): contiguous bounds
 * over n items with nonnegative work[i], bounds[0] = 0, bounds[world] = n,
 * bounds[r] = the first index whose work prefix (counting half of the item
 * itself) reaches r/world of the total; shards may be empty.  bounds has
 * world + 1 entries.  TUCKER_E_ARG on null pointers, n < 0 or world < 1. */
int tucker_shard_bounds(const double* work, int64_t n, int world, int64_t* bounds);

/* TUCKER_HOST_COLLECTIVES handles: fn is an
 *   int fn(void* dev_buf, int64_t count, int dtype, void* stream, void* user)
 * that replaces dev_buf (count elements, dtype 0 = fp32, 1 = fp64, device
 * memory of this rank) by its sum over the ranks and returns 0; the library
 * synchronises its stream before the call and the whole device after it (the
 * callback may write the result back on any stream).  Set it before the first sweep.
 * TUCKER_E_ARG for a handle without host collectives. */
int tucker_set_allreduce(tucker_handle* h, void* fn, void* user);

/* This rank's shards (out has 2 N + 2 N N entries): out[2n], out[2n + 1] =
 * [lo, hi) of the root slices of mode n's HOOI projection; out[2N + 2(nN + m)],
 * [.. + 1] = [lo, hi) of the slice index of MP term (n, m) (0, 0 for n == m).
 * Unsharded handles report the full ranges. */
int tucker_shard_info(tucker_handle* h, int64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* TUCKER_H */
