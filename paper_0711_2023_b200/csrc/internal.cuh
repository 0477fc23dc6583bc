// internal.cuh -- data structures and kernel entry points shared by the
// libtucker translation units.  See DESIGN.md for the layouts.
#pragma once

#include "common.cuh"

#include <memory>

namespace tk {

constexpr int kMaxOrder = 8;  // HOOI orders 2..8 (gen.cu for 2 and 5..8); MP / SP: 3, 4
constexpr int kMaxJ = 240;       // per-mode core size limit (eigensolver block k = J + p <= 256)
constexpr int kMaxJFused = 112;  // the persistent eigensolver's limit (block <= 116); larger J: eig_large
constexpr int kMaxBlock = 116;   // eigensolver block size k limit (Jacobi in shared memory)

// ---------------------------------------------------------------------------
// CSF: nonzeros sorted by (root, mid0[, mid1], leaf).
// sorts the COO file by mode n and writes one slice per index;
// here the sorted arrays stay in HBM and slice/fiber pointers replace files.
//   slice_ptr[r]..slice_ptr[r+1]   children of root index r: fibers (order 3)
//                                  or nodes (order 4)
//   node_ptr / node_mid0           order 4: runs of equal (root, mid0) -> fibers
//   fib_ptr[f]..fib_ptr[f+1]       nonzeros of fiber f (fixed root and mids)
//   fib_root, fib_mid0, fib_mid1   coordinates of fiber f
//   leaf_id, val                   per nonzero
// ---------------------------------------------------------------------------
struct Csf {
  int order = 0;
  int root = -1, mid0 = -1, mid1 = -1, leaf = -1;  // mode ids (0-based)
  int64_t I_root = 0, I_mid0 = 0, I_mid1 = 1, I_leaf = 0;
  int64_t nnz = 0, nfib = 0, nnode = 0;
  DBuf<int32_t> slice_ptr, node_ptr, node_mid0, fib_ptr, fib_root, fib_mid0, fib_mid1, leaf_id;
  DBuf<float> val;
  // HOOI SpTTMc work plan (order 3, spttmc_plan), built only for skewed
  // tensors: fibers longer than lmax nonzeros are cut into virtual fibers
  // (same mid index; Eq. 1 is linear in t_f), and slices whose work
  // J_l*nnz + J_m*J_l*fibers exceeds cmax are cut into units over virtual-
  // fiber ranges that write fp32 partial tiles, summed per slice in fixed
  // order (deterministic).  Units are ordered heaviest first so the block
  // scheduler packs them greedily.
  int64_t nunits = 0, nred = 0, nslots = 0, nvfib = 0, lmax = 0;
  double cmax = 0;
  DBuf<int32_t> vfib_ptr, vfib_mid;  // virtual fibers (nvfib + 1 / nvfib)
  DBuf<int32_t> unit;  // 4 ints per unit: slice, vf0, vf1, slot (-1: write Y directly)
  DBuf<int32_t> red;   // 3 ints per split slice: slice, first slot, #slots
  DBuf<float> part;    // nslots x (J_mid * J_leaf) partial tiles
  // order-4 GEMM-form SpTTMc (spttmc4g.cu): the ordering's "dense batch layout",
  // built on first use
  struct G4 {
    int nb_ = 0, kch = 0;              // nodes per batch, mid1 indices per chunk (0: not built)
    int64_t nbatch = 0;
    DBuf<int4> batch;                  // (slice, first node, nodes, -)
    DBuf<int32_t> bfirst, sp, tgt, leaf;  // first batch per slice; slot nonzero offsets (slots sorted by count per
                                          // chunk) and their (b_local, v) targets; leaf ids in slot order
    DBuf<float> val, part;             // values in slot order; run partial rows
    std::vector<int32_t> bfirst_h;
    // sibling-mode lists (HOOI partial-contraction reuse): nodes grouped by mid0
    bool sib_built = false;
    DBuf<int32_t> sib_ptr, sib_node, node_root;
  };
  std::unique_ptr<G4> g4 = std::make_unique<G4>();
};

struct Coo {  // validated, zero-free COO on the device
  int order = 0;
  int64_t dims[kMaxOrder] = {};
  int64_t nnz = 0;
  DBuf<int32_t> idx[kMaxOrder];
  DBuf<float> val;
};

// csf.cu
void coo_validate_compact(Coo& coo, cudaStream_t st);          // E_INDEX / E_VALUE, drops zeros
double coo_norm2(const Coo& coo, cudaStream_t st);              // ||X||_F^2 (fp64, fixed order)
void csf_build(const Coo& coo, Csf& out, int root, int mid0, int mid1, int leaf, cudaStream_t st);
// S += X_(n) X_(n)^T over the fibers [f0, f1) of an ordering whose leaf is n
// (S fp64, row stride lds, zeroed by the caller; both triangles written)
void sparse_gram(const Csf& c, int64_t f0, int64_t f1, double* S, int64_t lds, cudaStream_t st);
// spttmc.cu: HOOI work units for an order-3 CSF whose output tile is Jm x Jl
// (lo, hi): the rank's root-slice range (hi < 0: all)
void spttmc_plan(Csf& c, int64_t Jm, int64_t Jl, int num_sms, cudaStream_t st, int64_t lo = 0, int64_t hi = -1);

// ---------------------------------------------------------------------------
// Split-fp32 matrix: a = hi + lo exactly, hi = tf32-rounded a (DESIGN.md
// "3xTF32 operands").  Row-major rows x ld, zero padded.
// ---------------------------------------------------------------------------
struct Split {
  float* hi = nullptr;
  float* lo = nullptr;
  int64_t rows = 0, cols = 0, ld = 0;  // logical rows/cols; ld = padded row length
  // Gram K extent when the view covers part of each row (a K-range shard of
  // Y^T whose pointers are offset by a multiple of 32 columns); 0 = ld
  int64_t kext = 0;
  // K-tile-major layout (MP's W): element (r, c) at (c / 32) * 32 ld + 32 r + c % 32,
  // ld = rows rounded up to 8, kext = columns rounded up to 32.  Each 32-column K-tile
  // of a 128-row block is one contiguous 16 KB box for TMA.
  bool ktile = false;
  int64_t K() const { return kext > 0 ? kext : ld; }
};

// gen.cu: HOOI projection for orders 2 and 5..8 -- per mode n the nonzeros sorted by
// (i_n, other modes lower-fastest) as one 64-bit key, and the slice pointers of mode n
struct GenMode {
  DBuf<uint64_t> key;
  DBuf<float> val;
  DBuf<int32_t> sptr;  // I_n + 1
  int64_t nnz = 0;
  uint64_t Sn = 1;     // prod_{m != n} I_m
};
void gen_build(Coo& coo, GenMode* modes, cudaStream_t st);  // validates (E_INDEX, E_VALUE, E_DUP)
void spttmc_gen(const GenMode& g, int order, int n, const int64_t* dims, const int64_t* J, const float* const* U,
                Split Y, bool transposed, cudaStream_t st);


// spttmc.cu
// HOOI: Y_(n) (Kolda order) written as split fp32; transposed => out is Y_(n)^T.
// Only the root slices [lo, hi) are computed (a rank's shard; hi < 0: all); the
// other rows of out stay as they are (zero).
// order-4 GEMM-form SpTTMc (spttmc4g.cu); false: not applicable (use k_spttmc4w)
// zout (nullable): Z_v = U_mid1^T T_v of every node, [nnode][J_mid1 round_up(J_leaf, 4)], kept for
// the sibling mode (FMA kernel only)
bool spttmc4g(const Csf& c, const float* const* U, const int64_t* J, Split out, bool transposed, int64_t s0,
              int64_t s1, int64_t sb, cudaStream_t st, int64_t lo, int64_t hi, float* zout = nullptr);
bool spttmc4g_fma_default(const Csf& c, const int64_t* J);  // spttmc4g would run the FMA kernel by default
// Y_(c.mid0) from the kept Z of ordering c (strides: Kolda positions of root, mid1, leaf in mode mid0's unfolding)
void spttmc4_sibling(const Csf& c, const float* Z, const float* Uroot, const int64_t* J, Split out, bool transposed,
                     int64_t sr, int64_t s1, int64_t sb, cudaStream_t st);
void spttmc_hooi_sibling(const Csf& c, const float* Z, const float* const* U, const int64_t* J, Split out,
                         bool transposed, cudaStream_t st);
void spttmc_hooi(const Csf& c, const float* const* U, const int64_t* J, Split out, bool transposed,
                 cudaStream_t st, int64_t lo = 0, int64_t hi = -1, float* zout = nullptr);
// MP: W columns [col_off, col_off + (s_hi - s_lo)*J_leaf) of the rows of out
// (out pre-zeroed): W[i_root, col_off + (mk - s_lo)*J_leaf + j] = sum_{x in fiber} x U_leaf[i_leaf, j]
// for the slices mk (the mid index) in [s_lo, s_hi) (a rank's shard; s_hi < 0: all).
void spmm_mp(const Csf& c, const float* U_leaf, int64_t J_leaf, Split out, int64_t col_off,
             cudaStream_t st, int64_t s_lo = 0, int64_t s_hi = -1);

// dist.cu -- NCCL (loaded on demand) and shard bounds for the sharded sweep
void* dist_comm_init(const void* unique_id, int world, int rank);
void dist_comm_destroy(void* comm);
void* dist_comm_host();  // TUCKER_HOST_COLLECTIVES: sums through a host callback
void dist_comm_set_callback(void* comm, void* fn, void* user);
void dist_allreduce_f32(void* comm, float* p, int64_t n, cudaStream_t st);
void dist_allreduce_f64(void* comm, double* p, int64_t n, cudaStream_t st);
// rank r owns elements [off[r], off[r + 1]) of base (off has world + 1 entries); all ranks get all
void dist_allgatherv_f32(void* comm, float* base, const int64_t* off, int world, cudaStream_t st);
void dist_allgatherv_f64(void* comm, double* base, const int64_t* off, int world, cudaStream_t st);
void dist_unique_id(void* out128);
void shard_bounds(const double* w, int64_t n, int world, int64_t* bounds);

// gram.cu -- S (d x d fp64, row-major, ld = lds) = A A^T, A = d x K split fp32.
struct GramWs {
  DBuf<double> partial;
  DBuf<uint8_t> scratch;
};
// S = A A^T (+ Sadd, same layout, when given: the MP term split of mp_sweep's overlap);
// fma_hint > 0: choose the precision path by this size (the whole Gram a part belongs to)
void gram_syrk(const Split& A, double* S, int64_t lds, GramWs& ws, cudaStream_t st, const double* Sadd = nullptr,
               double fma_hint = 0);
// fp64 tensor-core (DMMA) path for Grams small enough to afford fp64
void gram_syrk_dmma(const Split& A, double* S, int64_t lds, GramWs& ws, cudaStream_t st, const double* Sadd = nullptr);
int gram_mode();     // 0 = by size (default), 1 = every Gram on fp64 DMMA (env TUCKER_GRAM_FP64=1)
int gram_path_id();  // 0 = by size (DMMA <= 2e10 FMA, else tcgen05 3xTF32), 1 = all DMMA

// dense.cu -- small fp64 dense kernels for the eigensolver and the core.
enum class Elt { F64, F32, SPLIT };
struct MatRef {
  Elt t = Elt::F64;
  const void* p = nullptr;     // F64: double*, F32: float*
  const float* lo = nullptr;   // SPLIT: p = hi, lo = lo
  int64_t ld = 0;
  bool trans = false;          // op(A) = A^T
};
struct DenseWs {
  DBuf<double> splitk;
};
// C (M x N fp64, ldc) = alpha op(A) op(B) + beta C + gamma D (D nullable, ldd)
void dgemm(int64_t M, int64_t N, int64_t K, double alpha, MatRef A, MatRef B, double beta,
           double* C, int64_t ldc, double gamma, const double* D, int64_t ldd, DenseWs& ws,
           cudaStream_t st);
// ... + delta E (E nullable, lde): the fused Chebyshev-recurrence epilogue
void dgemm4(int64_t M, int64_t N, int64_t K, double alpha, MatRef A, MatRef B, double beta,
            double* C, int64_t ldc, double gamma, const double* D, int64_t ldd, double delta,
            const double* E, int64_t lde, DenseWs& ws, cudaStream_t st);
double dnorm2_f32(const float* x, int64_t n, DenseWs& ws, cudaStream_t st);  // sum x^2, fp64

// eig.cu
struct EigSlot {              // warm-start state per (algorithm, mode)
  DBuf<double> basis;         // d x k Ritz vectors of the last solve (row-major)
  int64_t d = 0;
  int k = 0;
  bool valid = false;
  double lmin = 0.0, bval = 0.0;  // lambda_min estimate and filter bound of the last solve
  int lz_age = 0;                  // solves since the last Lanczos estimate
  int exact_age = 0;               // consecutive exact warm starts (no re-orthonormalisation)
};
struct EigWs {
  DBuf<double> Q, SQ, X, Y, T;  // eig_fused work blocks (padded layout)
  DBuf<double> L, LT, pq, py, pz;  // locked vectors, S L, power-iteration / Lanczos vectors
  DBuf<double> fpart, fred;     // eig_fused reduction partials / results
  DBuf<double> mpart;           // eig_fused split-K partial products
  DBuf<long long> fprof;        // eig_fused per-phase ns (accumulated over solves)
  bool fprof_init = false;
  DBuf<double> cq, ct, H, R;    // cholqr2 (Y^T Y route)
  DBuf<double> bL, bQ, bSQ, bY0, bY1, bT, sH, sV, sC, sTh, sRes;  // eig_large work blocks
  DBuf<int> sInfo;
  DBuf<double> small;  // eig_small scratch
  DenseWs dense;
  int64_t stat_outer = 0, stat_matvec = 0, stat_sweeps = 0;
};
struct EigOpts {
  int oversample = 0;
  int max_outer = 60;             // tucker_opts.eig_max_iter default (include/tucker.h)
  int jacobi_sweeps = 2;        // cap per Rayleigh-Ritz step (residuals decide convergence)
  int jacobi_sweeps_first = 1;  // cap for a solve's first Rayleigh-Ritz step (measured best at config 2)
  double tol = 1e-10;
};
// Leading J eigenvectors of symmetric PSD S (d x d in the padded layout of
// eig_layout: row stride ls, `rows` allocated rows; S is used as workspace and
// deflated in place) in one persistent cooperative kernel (eig_fused.cu):
// out_V (d x J, ld = J) and theta_dev (J, descending) on the device,
// info_dev[0..4] = {converged, outer iterations, matvecs, Jacobi sweeps,
// breakdown}.  No host synchronisation.
void eig_layout(int64_t d, int64_t* ls, int64_t* rows);
bool eig_fused(double* S, int64_t d, int J, EigSlot& slot, EigWs& ws, const EigOpts& o, double* out_V,
               double* theta_dev, int* info_dev, cudaStream_t st, const float* hint = nullptr);
size_t eig_fused_smem(int k, int d, int G);
// d > kFusedMaxD (the persistent solver keeps each CTA's rows of the block in shared
// memory): the same method as a host-driven kernel sequence (eig_large.cu); S row
// stride ls, same outputs and info record as eig_fused.  Synchronises the stream.
constexpr int64_t kFusedMaxD = 8192;
// Direct dense solver for d <= kSmallMaxD (eig_small.cu): Householder tridiagonalisation
// in one 4-CTA cluster, bisection + inverse iteration, back-transformation.  V (n x m,
// ld m), theta (m, descending), info record as eig_fused; scratch is a work buffer.
constexpr int64_t kSmallMaxD = 256;
void eig_small(const double* S, int64_t n, int64_t lds, int m, double* V, double* theta, int* info, DBuf<double>& scratch,
               cudaStream_t st);
// doubles of shared memory the one-CTA direct solver needs for (n, m); 0: it does not fit
size_t eig_direct_ws(int n, int m);
bool eig_large(const double* S, int64_t d, int64_t ls, int J, EigSlot& slot, EigWs& ws, const EigOpts& o,
               double* out_V, double* theta_dev, int* info_dev, cudaStream_t st, const float* hint = nullptr);
// MP's multislice Gram without the dense W (mp_sparse.cu): M (fp64, upper triangle, row
// stride ls) += sum over the slices [s_lo, s_hi) of the order-3 CSF c (root = the slice
// mode o, mid = n, leaf = m) of P_s P_s^T, P_s = X_s U_m; P rows are staged in Pbuf
// (at most max_p_floats floats per batch of slices).  mp_sparse_mirror fills the lower triangle.
void mp_sparse_term(const Csf& c, const float* U_leaf, int64_t J, int64_t s_lo, int64_t s_hi, double* M, int64_t ls,
                    DBuf<float>& Pbuf, size_t max_p_floats, cudaStream_t st);
void mp_sparse_mirror(double* M, int64_t d, int64_t ls, cudaStream_t st);
// unit test of the fused solver's k x k routines (one CTA); see tucker_debug_smalldense
void eig_unit_mv(const double* S, const double* Y, int d, int n, double alpha, double* Out, double gamma,
                 const double* D, cudaStream_t st);
double eig_unit_mv_time(int d, int n, int reps);  // us per product (zero data)
double eig_unit_mv_repeat(const double* S, const double* Y, int d, int n);
void eig_unit(int mode, const double* in, int k, double* out, double* theta, int* iout, int sweeps,
              double shift, cudaStream_t st);
// Orthonormalise the columns of V (d x J fp64) in place (CholQR2).
void cholqr2(double* V, int64_t ldv, int64_t d, int J, EigWs& ws, cudaStream_t st);
// Order-preserving sign canonicalisation + fp32 conversion: U[i*J+j] = s_j V[i*ldv+j].
void canon_to_f32(const double* V, int64_t ldv, int64_t d, int J, float* U, cudaStream_t st);

}  // namespace tk
