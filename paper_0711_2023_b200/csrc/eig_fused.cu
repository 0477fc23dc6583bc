// eig_fused.cu -- leading-J eigenvectors of a symmetric PSD fp64 matrix in ONE
// persistent cooperative kernel.
//
// Figs. 1-8 "A <- J leading eigenvectors of ..." (the paper calls MATLAB
// `eigs(M*M', J, 'lm')`, ARPACK; SURVEY reading A2 uses M itself).
// Method: block Chebyshev-filtered subspace iteration
// with block size k = J + p, locking + explicit deflation, an outlier
// power-lock, shifted CholQR between filter segments and a Rayleigh-Ritz step
// whose k x k eigenproblem is solved by a parallel cyclic Jacobi in shared
// memory.  The whole iteration -- including the control decisions (filter
// degree, bounds, locking, convergence) -- runs on the device: every CTA
// executes the same control program on the same reduced scalars, so there is
// no host round trip and one launch per solve.
//
// Work split (G CTAs, one per SM, grid-wide barriers between dependent steps):
//   * rows: CTA c owns rows [c*R, (c+1)*R) of every d-row block (R = ceil(d/G));
//     row-local steps (axpby, Q <- Q M, copies, deflation of S's rows) need no
//     barrier among themselves.
//   * S * Y: CTA c computes its own rows of the product (reads all of Y).
//   * k x k reductions (Q^T Q, Q^T S Q, Ritz residuals): per-CTA partials over
//     its rows, a distributed fixed-order sum (deterministic), then every CTA
//     loads the result and runs the small dense step (LDL^T-based CholQR
//     factor, Jacobi) REDUNDANTLY in its own shared memory -- no further
//     barrier, and the k x k result is where the row-local apply needs it.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace tk {
namespace {

constexpr int NT = 512;  // threads per CTA
constexpr int NW = NT / 32;

struct FusedArgs {
  double* S;  // d x d row-major (deflated in place)
  int d, J, k;
  double* blk[5];           // five d x k work blocks (roles rotate)
  double* L;                // d x J locked vectors
  double* LT;               // d x J  S L
  double* part;             // [G][k*k] reduction partials
  double* red;              // [k*k] reduced result
  double* pvec[2];          // power iteration vectors (d)
  double* basis;            // d x k warm-start basis (read if warm, always written)
  int warm;
  double* outV;             // d x J output (ld = J)
  double* theta_out;        // J
  long long* prof;          // [8] per-phase ns (CTA 0's view), accumulated
  int* info;                // [0] converged [1] outer [2] matvecs [3] jacobi sweeps [4] breakdown
  double tol;
  int max_outer, jsweeps;
  uint64_t seed;
  int dbg;
  int noshift;
  int nolock;
  int nodefl;
};

// region 1 holds a k x (k+1) matrix or the own-row staging of a d x k block
__host__ __device__ inline size_t region1_doubles(int kp, int R) {
  const size_t a = (size_t)kp * (kp + 1), b = (size_t)R * kp;
  return a > b ? a : b;
}

struct Ctx {
  int cta, G, tid, warp, lane;
  int d, r0, r1;  // own rows [r0, r1)
  double* r1s;    // smem region 1 (k x (k+1) doubles or staging)
  double* r2s;    // smem region 2 (k x (k+1) doubles)
  size_t reg_doubles;
};

__device__ __forceinline__ void gsync() { cg::this_grid().sync(); }

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
enum { PF_MV = 0, PF_RED, PF_CHOL, PF_JAC, PF_APPLY, PF_DEFL, PF_POW, PF_OTHER };

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// ------------------------------------------------------------ row-local ops --
__device__ void copy_cols(const Ctx& x, const double* src, int lds, double* dst, int ldd, int ncol) {
  for (int r = x.r0 + x.warp; r < x.r1; r += NW)
    for (int c = x.lane; c < ncol; c += 32) dst[(int64_t)r * ldd + c] = src[(int64_t)r * lds + c];
}

__device__ void fill_random(const Ctx& x, double* Q, int k, uint64_t seed) {
  for (int r = x.r0 + x.warp; r < x.r1; r += NW)
    for (int c = x.lane; c < k; c += 32) {
    const uint64_t h = mix64(seed ^ mix64((uint64_t)r * 1315423911ull + (uint64_t)c));
    Q[(int64_t)r * k + c] = ((double)(h >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
  }
}

// z = a x + b y on own rows (ld = n), z may alias x or y
__device__ void axpby(const Ctx& x, int n, double a, const double* X, double b, const double* Y,
                      double* Z) {
  for (int r = x.r0 + x.warp; r < x.r1; r += NW)
    for (int c = x.lane; c < n; c += 32) {
      const int64_t o = (int64_t)r * n + c;
      Z[o] = a * X[o] + (b != 0.0 ? b * Y[o] : 0.0);
    }
}

// Out[own rows][0..n) = In[own rows][0..m) * M, M(l, c) from shared memory:
//   mode 0: M(l, c) = Ms[l * ldm + c]
//   mode 1: M(l, c) = Ms[perm[c] * ldm + l]   (Jacobi: rows of W are eigenvectors)
// In rows are staged in `stage` (own rows x m) first, so Out may alias In.
__device__ void apply_right(const Ctx& x, const double* In, int ldi, int m, const double* Ms, int ldm,
                            int mode, const int* perm, double* Out, int ldo, int n, double* stage) {
  const int nr = x.r1 - x.r0;
  if (nr <= 0) return;
  for (int r = x.warp; r < nr; r += NW)
    for (int l = x.lane; l < m; l += 32) stage[r * m + l] = In[(int64_t)(x.r0 + r) * ldi + l];
  __syncthreads();
  const int nch = (n + 31) >> 5;
  for (int t = x.warp; t < nr * nch; t += NW) {
    const int r = t / nch, c = ((t - r * nch) << 5) + x.lane;
    if (c >= n) continue;
    const double* a = stage + r * m;
    double s = 0.0;
    if (mode == 0) {
#pragma unroll 4
      for (int l = 0; l < m; ++l) s = fma(a[l], Ms[l * ldm + c], s);
    } else {
      const double* w = Ms + perm[c] * ldm;
#pragma unroll 4
      for (int l = 0; l < m; ++l) s = fma(a[l], w[l], s);
    }
    Out[(int64_t)(x.r0 + r) * ldo + c] = s;
  }
  __syncthreads();
}

// ------------------------------------------------- S * Y on the fp64 tensor cores --
// Out = alpha S Y + gamma D + delta E  (S d x d, Y/Out/D/E d x n, ld n; n <= 128).
// 2D tiling: CTA (rb, cb) computes rows [8 m8 rb, +8 m8) x column tiles [tpb cb, +tpb)
// of 8 columns; the plan (m8, CB) minimises max(DMMA time, L2 traffic time) over
// the G CTAs and is computed identically by every CTA.  K is staged in chunks of
// KCH through shared memory with cp.async (double buffered, zero-filled edges);
// warp w owns n-tile pair (w mod ng) for every row tile and the k4-steps
// congruent to (w / ng) mod KS; the KS partial tiles are summed in a fixed
// order in the epilogue.  mma.sync m8n8k4 f64 -> DMMA on sm_100a.
// Y must be complete (barrier before); Out must not alias Y; E may alias Y.
constexpr int KCH = 64;          // K per staged chunk (16 k4-steps)
constexpr int SP = KCH + 4;      // S tile row stride (conflict-free A fragments)
constexpr int M8MAX = 6;         // row tiles per CTA
constexpr int NSMAX = 4;         // pipeline stages
constexpr size_t MV_BUDGET = 200 * 1024 / sizeof(double);  // doubles of smem for the stages

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  const int nbytes = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "r"(nbytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct MvPlan {
  int m8, CB, tpb, RBn;
};
__host__ __device__ inline MvPlan mv_plan(int d, int n, int G) {
  const int n8 = (n + 7) >> 3;
  MvPlan best{1, 1, n8, (d + 7) >> 3};
  double bt = 1e300;
  for (int m8 = 1; m8 <= M8MAX; ++m8) {
    const int RBn = (d + 8 * m8 - 1) / (8 * m8);
    for (int CB = 1; CB <= n8; ++CB) {
      const int tpb = (n8 + CB - 1) / CB;
      const int cbn = (n8 + tpb - 1) / tpb;
      if (cbn != CB || RBn * cbn > G) continue;
      const double comp = 64.0 * m8 * tpb * (double)d / 64.0;                        // clk at ~64 FMA/clk
      const double traf = (double)RBn * cbn * 8.0 * (m8 + tpb) * 8.0 * d / 6000.0;   // clk at ~6 KB/clk L2
      const double t = comp > traf ? comp : traf;
      if (t < bt - 1e-9) {
        bt = t;
        best = MvPlan{m8, cbn, tpb, RBn};
      }
    }
  }
  return best;
}
__host__ __device__ inline int mv_ypad(int tpb) { return ((8 * tpb + 15) & ~15) + 4; }
__host__ __device__ inline size_t mv_stage_doubles(int m8, int tpb) {
  return (size_t)8 * m8 * SP + (size_t)KCH * mv_ypad(tpb);
}
__host__ __device__ inline int mv_stages(int m8, int tpb) {
  const size_t st = mv_stage_doubles(m8, tpb);
  int ns = (int)(MV_BUDGET / st);
  return ns > NSMAX ? NSMAX : (ns < 2 ? 2 : ns);
}
__host__ __device__ inline size_t mv_smem_doubles(int m8, int tpb) {
  return (size_t)mv_stages(m8, tpb) * mv_stage_doubles(m8, tpb);
}

// ------------------------------------------------- S * Y on the fp64 tensor cores --
// Out = alpha S Y + gamma D + delta E  (S d x d, Y/Out/D/E d x n, ld n; n <= 128).
// 2D tiling: CTA (rb, cb) computes rows [8 m8 rb, +8 m8) x column tiles [tpb cb, +tpb)
// of 8 columns; the plan (m8, CB) minimises max(DMMA time, L2 traffic time) over
// the G CTAs and is computed identically by every CTA.  K is streamed in chunks
// of KCH through an NS-stage cp.async pipeline (zero-filled edges, one barrier per
// chunk); warp w owns n-tile pair (w mod ng) for every row tile and the k4-steps
// congruent to (w / ng) mod KS; the KS partial tiles are summed in a fixed order
// in the epilogue.  mma.sync m8n8k4 f64 -> DMMA on sm_100a.
// Y must be complete (barrier before); Out must not alias Y, D; E may alias Y.
// the plan of mv_plan(), evaluated with one candidate (m8, CB) per thread and a
// block-wide argmin (same tie-break: smallest m8, then smallest CB); cached per n
__device__ MvPlan mv_plan_cached(const Ctx& x, int n) {
  __shared__ int cn, init;
  __shared__ MvPlan cpl;
  __shared__ double bt[NW];
  __shared__ int bi[NW];
  if (init == 0x5eed && cn == n) {
    const MvPlan p = cpl;
    __syncthreads();
    return p;
  }
  __syncthreads();
  const int d = x.d;
  const int n8 = (n + 7) >> 3;
  double t = 1e300;
  int id = 1 << 30;
  if (x.tid < M8MAX * n8) {
    const int m8 = 1 + x.tid / n8, CB = 1 + x.tid % n8;
    const int RBn = (d + 8 * m8 - 1) / (8 * m8);
    const int tpb = (n8 + CB - 1) / CB;
    const int cbn = (n8 + tpb - 1) / tpb;
    if (cbn == CB && RBn * cbn <= x.G) {
      const double comp = 64.0 * m8 * tpb * (double)d / 64.0;
      const double traf = (double)RBn * cbn * 8.0 * (m8 + tpb) * 8.0 * d / 6000.0;
      t = comp > traf ? comp : traf;
      id = x.tid;
    }
  }
  // argmin with the serial loop's preference for the first candidate within 1e-9
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ot = __shfl_xor_sync(0xffffffffu, t, o);
    const int oi = __shfl_xor_sync(0xffffffffu, id, o);
    if (ot < t - 1e-9 || (fabs(ot - t) <= 1e-9 && oi < id)) {
      t = ot;
      id = oi;
    }
  }
  if (x.lane == 0) {
    bt[x.warp] = t;
    bi[x.warp] = id;
  }
  __syncthreads();
  if (x.tid == 0) {
    double b = 1e300;
    int ib = 1 << 30;
    for (int w = 0; w < NW; ++w)
      if (bt[w] < b - 1e-9 || (fabs(bt[w] - b) <= 1e-9 && bi[w] < ib)) {
        b = bt[w];
        ib = bi[w];
      }
    MvPlan p{1, 1, n8, (d + 7) >> 3};
    if (ib < (1 << 30)) {
      const int m8 = 1 + ib / n8, CB = 1 + ib % n8;
      const int tpb = (n8 + CB - 1) / CB;
      p = MvPlan{m8, CB, tpb, (d + 8 * m8 - 1) / (8 * m8)};
    }
    cpl = p;
    cn = n;
    init = 0x5eed;
  }
  __syncthreads();
  const MvPlan p = cpl;
  __syncthreads();
  return p;
}

__device__ void matvec(const Ctx& x, const double* S, const double* Y, int n, double alpha, double* Out,
                       double gamma, const double* Dm, double delta, const double* Em) {
  const int d = x.d;
  const MvPlan pl = mv_plan_cached(x, n);
  if (x.cta >= pl.RBn * pl.CB) return;
  const int rb = x.cta / pl.CB, cb = x.cta - rb * pl.CB;
  const int MT = 8 * pl.m8;
  const int row0 = rb * MT;
  const int n8 = (n + 7) >> 3;
  const int t0 = cb * pl.tpb;
  const int ntile = min(pl.tpb, n8 - t0);
  if (row0 >= d || ntile <= 0) return;
  const int col0 = 8 * t0;
  const int NTL = 8 * ntile;
  const int YP = mv_ypad(pl.tpb);
  const int NS = mv_stages(pl.m8, pl.tpb);
  const size_t STG = mv_stage_doubles(pl.m8, pl.tpb);
  const int ng = (ntile + 1) >> 1;  // n-tile pairs
  const int KS = NW / ng;           // >= 2 (ntile <= 16)
  const int myg = x.warp % ng, myks = x.warp / ng;
  const bool wact = myks < KS;
  const int nt0 = 2 * myg;
  const bool two = nt0 + 1 < ntile;
  double acc[M8MAX][2][2];
#pragma unroll
  for (int i = 0; i < M8MAX; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto stage = [&](int ch) {
    double* sS = x.r1s + (size_t)(ch % NS) * STG;
    double* sY = sS + MT * SP;
    const int k0 = ch * KCH;
    for (int r = x.warp; r < MT; r += NW) {
      const int gr = row0 + r;
#pragma unroll
      for (int h = 0; h < KCH / 32; ++h) {
        const int kk = x.lane + 32 * h;
        const bool ok = gr < d && k0 + kk < d;
        cp_async8(sS + r * SP + kk, ok ? S + (int64_t)gr * d + k0 + kk : S, ok);
      }
    }
    for (int kk = x.warp; kk < KCH; kk += NW) {
      const int gk = k0 + kk;
      for (int c = x.lane; c < NTL; c += 32) {
        const bool ok = gk < d && col0 + c < n;
        cp_async8(sY + kk * YP + c, ok ? Y + (int64_t)gk * n + col0 + c : Y, ok);
      }
    }
  };
  const int nch = (d + KCH - 1) / KCH;
  // prologue: NS - 1 chunks in flight (empty groups keep the accounting uniform)
  for (int ch = 0; ch < NS - 1; ++ch) {
    if (ch < nch) stage(ch);
    cp_commit();
  }
  const int ar = x.lane >> 2, aq = x.lane & 3;  // fragment coordinates
  for (int ch = 0; ch < nch; ++ch) {
    if (NS == 4) cp_wait<2>();
    else if (NS == 3) cp_wait<1>();
    else cp_wait<0>();
    __syncthreads();  // chunk ch visible to all; buffer (ch - 1) % NS free
    if (ch + NS - 1 < nch) stage(ch + NS - 1);
    cp_commit();
    if (wact) {
      const double* sS = x.r1s + (size_t)(ch % NS) * STG;
      const double* sY = sS + MT * SP;
      for (int s4 = myks; s4 < KCH / 4; s4 += KS) {
        const int kb = 4 * s4;
        const double b0 = sY[(kb + aq) * YP + 8 * nt0 + ar];
        const double b1 = two ? sY[(kb + aq) * YP + 8 * (nt0 + 1) + ar] : 0.0;
#pragma unroll
        for (int i = 0; i < M8MAX; ++i) {
          if (i < pl.m8) {
            const double a = sS[(8 * i + ar) * SP + kb + aq];
            dmma(acc[i][0][0], acc[i][0][1], a, b0);
            if (two) dmma(acc[i][1][0], acc[i][1][1], a, b1);
          }
        }
      }
    }
  }
  cp_wait<0>();
  __syncthreads();
  // epilogue: partial tiles -> smem [KS][MT][NTL], fixed-order sum over KS
  double* red = x.r1s;
  if (wact) {
#pragma unroll
    for (int i = 0; i < M8MAX; ++i) {
      if (i < pl.m8) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (j == 0 || two) {
            const int rr = 8 * i + ar, cc = 8 * (nt0 + j) + 2 * aq;
            double* o = red + ((size_t)myks * MT + rr) * NTL + cc;
            o[0] = acc[i][j][0];
            o[1] = acc[i][j][1];
          }
        }
      }
    }
  }
  __syncthreads();
  const int nrow = min(MT, d - row0);
  const int ncol = min(NTL, n - col0);
  for (int r = x.warp; r < nrow; r += NW)
    for (int c = x.lane; c < ncol; c += 32) {
      double sum = 0.0;
      for (int q = 0; q < KS; ++q) sum += red[((size_t)q * MT + r) * NTL + c];
      const int64_t o = (int64_t)(row0 + r) * n + col0 + c;
      double v = alpha * sum;
      if (gamma != 0.0) v += gamma * Dm[o];
      if (delta != 0.0) v += delta * Em[o];
      Out[o] = v;
    }
  __syncthreads();
}

// single vector: y[own rows] = S[own rows, :] q, partial ||y||^2 -> part[cta]
__device__ void matvec1(const Ctx& x, const double* S, const double* q, double* y,
                        double* part) {
  __shared__ double wsum[NW];
  double nrm = 0.0;
  for (int r = x.r0 + x.warp; r < x.r1; r += NW) {
    const double* srow = S + (int64_t)r * x.d;
    double s = 0.0;
    for (int c = x.lane; c < x.d; c += 32) s = fma(__ldcg(srow + c), __ldcg(q + c), s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (x.lane == 0) y[r] = s;
    nrm = fma(s, s, nrm);  // lane 0 carries the row's value
  }
  if (x.lane == 0) wsum[x.warp] = nrm;
  __syncthreads();
  if (x.tid == 0) {
    double t = 0.0;
    for (int w = 0; w < NW; ++w) t += wsum[w];
    part[x.cta] = t;
  }
  __syncthreads();
}

// every CTA: sum of part[0..G) in a fixed order (after a barrier)
__device__ double allsum_scalar(const Ctx& x, const double* part) {
  __shared__ double res;
  if (x.warp == 0) {
    double s = 0.0;
    for (int z = x.lane; z < x.G; z += 32) s += __ldcg(part + z);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (x.lane == 0) res = s;
  }
  __syncthreads();
  const double r = res;
  __syncthreads();
  return r;
}

// every CTA: max over CTAs of a per-thread value (debug diagnostics)
__device__ double gmax(const Ctx& x, double v, double* part) {
  __shared__ double wm[NW];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (x.lane == 0) wm[x.warp] = v;
  __syncthreads();
  if (x.tid == 0) {
    double m = 0.0;
    for (int w = 0; w < NW; ++w) m = fmax(m, wm[w]);
    part[x.cta] = m;
  }
  __syncthreads();
  gsync();
  __shared__ double res;
  if (x.tid == 0) {
    double m = 0.0;
    for (int z = 0; z < x.G; ++z) m = fmax(m, __ldcg(part + z));
    res = m;
  }
  __syncthreads();
  const double r = res;
  gsync();
  return r;
}

// ------------------------------------------------------- k x k reductions --
// part[cta][i*nb + j] = sum_{own rows r} A[r][i] B[r][j]
__device__ void gram_partial(const Ctx& x, const double* A, int lda, int na, const double* B, int ldb,
                             int nb, double* part) {
  const int nr = x.r1 - x.r0;
  const int E = na * nb;
  double* sA = x.r1s;
  double* sB = x.r1s + (size_t)nr * na;
  for (int r = x.warp; r < nr; r += NW) {
    for (int c = x.lane; c < na; c += 32) sA[r * na + c] = A[(int64_t)(x.r0 + r) * lda + c];
    for (int c = x.lane; c < nb; c += 32) sB[r * nb + c] = B[(int64_t)(x.r0 + r) * ldb + c];
  }
  __syncthreads();
  double* out = part + (size_t)x.cta * E;
  for (int i = x.warp; i < na; i += NW)
    for (int j = x.lane; j < nb; j += 32) {
      double s = 0.0;
      for (int r = 0; r < nr; ++r) s = fma(sA[r * na + i], sB[r * nb + j], s);
      out[i * nb + j] = s;
    }
  __syncthreads();
}

// red[e] = sum_z part[z][e] (fixed order), entries distributed over CTAs; then
// barrier and every CTA copies red into dst (smem, row stride ldd, nb columns).
__device__ void reduce_bcast(const Ctx& x, const double* part, int E, int nb, double* red, double* dst,
                             int ldd) {
  gsync();
  const int per = (E + x.G - 1) / x.G;
  const int e0 = x.cta * per, e1 = min(E, e0 + per);
  // 8 threads per entry, each a strided subset of the partials, combined by shuffles
  for (int base = e0; base < e1; base += NT / 8) {
    const int e = base + x.tid / 8, sub = x.tid % 8;
    double s = 0.0;
    if (e < e1)
      for (int z = sub; z < x.G; z += 8) s += __ldcg(part + (size_t)z * E + e);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    if (e < e1 && sub == 0) red[e] = s;
  }
  gsync();
  const int nrow = E / nb;
  for (int i = x.warp; i < nrow; i += NW)
    for (int j = x.lane; j < nb; j += 32) dst[i * ldd + j] = __ldcg(red + i * nb + j);
  __syncthreads();
}

// ---------------------------------------------------------- CholQR factor --
// G (k x k, in A = smem, ld) SPD.  Equilibrate (D G D + shift I, D = diag^-1/2)
// and eliminate symmetrically on [A | E] (E = I): after step j rows l > j of
// the upper part are reduced and E accumulates L^{-1} (G = L P L^T, P the
// pivots).  Then M = D E^T P^{-1/2} (upper triangular) satisfies M^T G M = I,
// written to X (smem, ld): Q M has orthonormal columns (CholQR).  One barrier
// per elimination step.
__device__ void cholqr_factor(const Ctx& x, double* A, double* X, int k, int ld, double shift) {
  __shared__ double dsc[kMaxBlock];
  for (int i = x.tid; i < k; i += NT) {
    const double g = A[i * ld + i];
    dsc[i] = g > 0 ? rsqrt(g) : 1.0;
  }
  __syncthreads();
  for (int r = x.warp; r < k; r += NW)
    for (int c = x.lane; c < k; c += 32) {
      A[r * ld + c] = A[r * ld + c] * dsc[r] * dsc[c] + (r == c ? shift : 0.0);
      X[r * ld + c] = (r == c) ? 1.0 : 0.0;
    }
  __syncthreads();
  for (int j = 0; j < k - 1; ++j) {
    const double pj = A[j * ld + j];
    const double ip = 1.0 / (pj > 1e-12 ? pj : 1e-12);
    // rows l > j, one warp per row: upper part (m >= l) and E part (m <= j)
    for (int l = j + 1 + x.warp; l < k; l += NW) {
      const double f = A[j * ld + l] * ip;
      double* al = A + l * ld;
      const double* aj = A + j * ld;
      for (int m = l + x.lane; m < k; m += 32) al[m] = fma(-f, aj[m], al[m]);
      double* el = X + l * ld;
      const double* ej = X + j * ld;
      for (int m = x.lane; m <= j; m += 32) el[m] = fma(-f, ej[m], el[m]);
    }
    __syncthreads();
  }
  // X <- M = D E^T P^{-1/2}: M[m][i] = dsc[m] E[i][m] / sqrt(P_i) for m <= i (upper
  // triangular), built in A (only A's diagonal -- the pivots -- is still needed).
  __shared__ double piv[kMaxBlock];
  for (int i = x.tid; i < k; i += NT) {
    const double p = A[i * ld + i];
    piv[i] = rsqrt(p > 1e-12 ? p : 1e-12);
  }
  __syncthreads();
  for (int m = x.warp; m < k; m += NW)
    for (int i = x.lane; i < k; i += 32) A[m * ld + i] = (m <= i) ? dsc[m] * X[i * ld + m] * piv[i] : 0.0;
  __syncthreads();
  for (int r = x.warp; r < k; r += NW)
    for (int c = x.lane; c < k; c += 32) X[r * ld + c] = A[r * ld + c];
  __syncthreads();
}

// ----------------------------------------------------------------- Jacobi --
// Parallel cyclic Jacobi on H (k x k, smem, ld = kp + 1 with kp = k + (k & 1)).
// Round r of a sweep pairs (kp-1, r) and ((r+i) mod (kp-1), (r-i) mod (kp-1)),
// i = 1..kp/2-1 (circle method); the kp/2 rotations of a round are disjoint.
// Per round: [rotation + rows of H and W] barrier [columns of H] barrier.
// The rotation angle is computed in fp32 (only its accuracy, not the
// orthogonality of the transform, depends on it: c = rsqrt(1 + t^2) and s = t c
// are formed in fp64).  W accumulates V^T (row i = eigenvector i).
// On exit theta (smem) holds the eigenvalues in descending order and perm[c]
// the row of W holding eigenvector c.  Returns the sweeps used (-1: non-finite).
__device__ int jacobi(const Ctx& x, double* H, double* W, int kin, int max_sweeps, double tol,
                      double* theta, int* perm) {
  const int kp = kin + (kin & 1);
  const int ld = kp + 1;
  const int np = kp / 2;
  __shared__ double cs_c[kMaxBlock / 2 + 1], cs_s[kMaxBlock / 2 + 1];
  __shared__ int pp[kMaxBlock / 2 + 1], pq[kMaxBlock / 2 + 1];
  __shared__ int bad;
  (void)0;
  // dummy index for odd k: zero coupling, -inf diagonal (sorts last)
  if (kin & 1) {
    for (int i = x.tid; i < kp; i += NT) {
      H[kin * ld + i] = (i == kin) ? -1e300 : 0.0;
      H[i * ld + kin] = (i == kin) ? -1e300 : 0.0;
    }
  }
  for (int r = x.warp; r < kp; r += NW)
    for (int c = x.lane; c < kp; c += 32) W[r * ld + c] = (r == c) ? 1.0 : 0.0;
  __syncthreads();
  const double tol2 = tol * tol;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    int any_sweep = 0;
    for (int round = 0; round < kp - 1; ++round) {
      int my_act = 0;
      // lane i of warp w computes the rotation of pair P = w + NW i (fp64), then the
      // warp applies its pairs' row updates
      const int npw = x.warp < np ? (np - x.warp + NW - 1) / NW : 0;
      int p = 0, q = 0;
      double c = 1.0, s = 0.0;
      if (x.lane < npw) {
        const int P = x.warp + NW * x.lane;
        if (P == 0) {
          p = kp - 1;
          q = round;
        } else {
          p = (round + P) % (kp - 1);
          q = (round - P + (kp - 1)) % (kp - 1);
        }
        const double app = H[p * ld + p], aqq = H[q * ld + q], apq = H[p * ld + q];
        if (apq != 0.0 && apq * apq > tol2 * fabs(app * aqq)) {
          const double tau = (aqq - app) / (2.0 * apq);
          const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(fma(tau, tau, 1.0)));
          c = 1.0 / sqrt(fma(t, t, 1.0));
          s = t * c;
        }
        cs_c[P] = c;
        cs_s[P] = s;
        pp[P] = p;
        pq[P] = q;
      }
      for (int i = 0; i < npw; ++i) {
        const double ci = __shfl_sync(0xffffffffu, c, i);
        const double si = __shfl_sync(0xffffffffu, s, i);
        const int pi = __shfl_sync(0xffffffffu, p, i);
        const int qi = __shfl_sync(0xffffffffu, q, i);
        if (si == 0.0) continue;
        my_act = 1;
        double* hp = H + pi * ld;
        double* hq = H + qi * ld;
        double* wp = W + pi * ld;
        double* wq = W + qi * ld;
        for (int j = x.lane; j < kp; j += 32) {
          const double a = hp[j], b = hq[j];
          hp[j] = ci * a - si * b;
          hq[j] = si * a + ci * b;
          const double u = wp[j], v = wq[j];
          wp[j] = ci * u - si * v;
          wq[j] = si * u + ci * v;
        }
      }
      const int any = __syncthreads_or(my_act);
      if (!any) continue;
      any_sweep = 1;
      // columns p, q of H for every pair: item = (pair, row)
      for (int P = x.warp; P < np; P += NW) {
        const double s = cs_s[P];
        if (s == 0.0) continue;
        const double c = cs_c[P];
        const int p = pp[P], q = pq[P];
        for (int i = x.lane; i < kp; i += 32) {
          const double a = H[i * ld + p], b = H[i * ld + q];
          H[i * ld + p] = c * a - s * b;
          H[i * ld + q] = s * a + c * b;
        }
      }
      __syncthreads();
    }
    if (!any_sweep) break;
  }
  // sort descending (stable by index)
  if (x.tid == 0) bad = 0;
  __syncthreads();
  if (x.tid < kp && !isfinite(H[x.tid * ld + x.tid]) && x.tid < kin) bad = 1;
  __syncthreads();
  if (x.tid < kp) {
    const double dv = H[x.tid * ld + x.tid];
    int rank = 0;
    for (int j = 0; j < kp; ++j) {
      const double e = H[j * ld + j];
      rank += (e > dv) || (e == dv && j < x.tid);
    }
    perm[rank] = x.tid;
  }
  __syncthreads();
  if (x.tid < kin) theta[x.tid] = H[perm[x.tid] * ld + perm[x.tid]];
  __syncthreads();
  const int r = bad ? -1 : sweep;
  __syncthreads();
  return r;
}

// -------------------------------------------------------------- the solver --
__global__ void __launch_bounds__(NT, 1) k_eig_fused(FusedArgs P) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double th[kMaxBlock + 2];    // Ritz values of the active block (indices nlock..)
  __shared__ double rs[kMaxBlock + 2];    // residuals
  __shared__ double thl[kMaxJ + 2];       // locked Ritz values
  __shared__ int perm[kMaxBlock + 2];

  Ctx x;
  x.cta = blockIdx.x;
  x.G = gridDim.x;
  x.tid = threadIdx.x;
  x.warp = x.tid >> 5;
  x.lane = x.tid & 31;
  x.d = P.d;
  const int d = P.d, J = P.J, k = P.k;
  const int R = (d + x.G - 1) / x.G;
  x.r0 = min(d, x.cta * R);
  x.r1 = min(d, x.r0 + R);
  const int kp = k + (k & 1);
  const int ld = kp + 1;
  x.r1s = smem;
  x.r2s = smem + region1_doubles(kp, R);
  double* S = P.S;

  // buffer roles (indices into P.blk), swapped identically by every CTA
  int iQ = 0, iSQ = 1, iX = 2, iY = 3, iT = 4;
  auto B = [&](int i) { return P.blk[i]; };

  int nlock = 0, ka = k;
  int n_rr = 0, matvecs = 0, jsw = 0, breakdown = 0;
  __shared__ long long pacc[8];
  long long pt = 0;
  if (x.tid < 8) pacc[x.tid] = 0;
  if (x.tid == 0) pt = gtimer();
  auto tick = [&](int cat) {
    if (x.cta == 0 && x.tid == 0) {
      const long long now = gtimer();
      pacc[cat] += now - pt;
      pt = now;
    }
  };

  if (P.warm) copy_cols(x, P.basis, k, B(iQ), k, k);
  else fill_random(x, B(iQ), k, P.seed);
  __syncthreads();

  // ---- orthonormalise the active block (ld = ka) against L and itself
  auto orth_active = [&](int passes, bool project) {
    if (nlock > 0 && project) {
      for (int pass = 0; pass < 2; ++pass) {
        gram_partial(x, P.L, J, nlock, B(iQ), ka, ka, P.part);
        reduce_bcast(x, P.part, nlock * ka, ka, P.red, x.r2s, ka);
        tick(PF_RED);
        // Q[own] -= L[own] Z  (Z = r2s, nlock x ka, ld ka)
        for (int r = x.r0 + x.warp; r < x.r1; r += NW)
          for (int c = x.lane; c < ka; c += 32) {
          double s = 0.0;
          for (int l = 0; l < nlock; ++l) s = fma(P.L[(int64_t)r * J + l], x.r2s[l * ka + c], s);
          B(iQ)[(int64_t)r * ka + c] -= s;
        }
        __syncthreads();
      }
    }
    const double shift = 11.0 * ((double)d * ka + (double)ka * (ka + 1)) * 1.1e-16 * ka;
    for (int pass = 0; pass < passes; ++pass) {
      gram_partial(x, B(iQ), ka, ka, B(iQ), ka, ka, P.part);
      reduce_bcast(x, P.part, ka * ka, ka, P.red, x.r1s, ld);
      tick(PF_RED);
      cholqr_factor(x, x.r1s, x.r2s, ka, ld, (pass == 0 && !P.noshift) ? shift : 0.0);
      tick(PF_CHOL);
      // stage rows in the tail of region 1 beyond the k x k block? region 1 is free now
      apply_right(x, B(iQ), ka, ka, x.r2s, ld, 0, nullptr, B(iQ), ka, ka, x.r1s);
      tick(PF_APPLY);
    }
  };

  // ---- Rayleigh-Ritz on the active block: Q <- Q V, SQ <- S Q V, th, rs
  auto rayleigh_ritz = [&]() {
    gsync();  // Q complete
    matvec(x, S, B(iQ), ka, 1.0, B(iSQ), 0.0, nullptr, 0.0, nullptr);
    gsync();  // SQ complete (the product is tiled, not row-local)
    tick(PF_MV);
    ++matvecs;
    gram_partial(x, B(iQ), ka, ka, B(iSQ), ka, ka, P.part);
    reduce_bcast(x, P.part, ka * ka, ka, P.red, x.r1s, ka + (ka & 1) + 1);
    tick(PF_RED);
    {
      const int kk = ka + (ka & 1);
      // symmetrise
      for (int r = x.warp; r < ka; r += NW)
        for (int c = x.lane; c < ka; c += 32) {
        if (r < c) {
          const double v = 0.5 * (x.r1s[r * (kk + 1) + c] + x.r1s[c * (kk + 1) + r]);
          x.r1s[r * (kk + 1) + c] = v;
          x.r1s[c * (kk + 1) + r] = v;
        }
      }
      __syncthreads();
      const int sw = jacobi(x, x.r1s, x.r2s, ka, k == d ? 60 : (n_rr == 0 ? P.jsweeps + 1 : P.jsweeps),
                            k == d ? 1e-15 : 1e-13, th + nlock, perm);
      tick(PF_JAC);
      if (sw < 0) breakdown = 1;
      else jsw += sw;
      ++n_rr;
      // Q <- Q V, SQ <- SQ V (V(l, c) = W[perm[c]][l]); staging in region 1 (H is dead)
      apply_right(x, B(iQ), ka, ka, x.r2s, kk + 1, 1, perm, B(iQ), ka, ka, x.r1s);
      tick(PF_APPLY);
      apply_right(x, B(iSQ), ka, ka, x.r2s, kk + 1, 1, perm, B(iSQ), ka, ka, x.r1s);
      tick(PF_APPLY);
    }
    // residual partials
    {
      const int nr = x.r1 - x.r0;
      double* out = P.part + (size_t)x.cta * ka;
      for (int c = x.tid; c < ka; c += NT) {
        const double t = th[nlock + c];
        double s = 0.0;
        for (int r = 0; r < nr; ++r) {
          const int64_t o = (int64_t)(x.r0 + r) * ka + c;
          const double v = B(iSQ)[o] - t * B(iQ)[o];
          s = fma(v, v, s);
        }
        out[c] = s;
      }
    }
    reduce_bcast(x, P.part, ka, ka, P.red, rs + nlock, ka);
    tick(PF_RED);
    for (int c = x.tid; c < ka; c += NT) rs[nlock + c] = sqrt(rs[nlock + c]);
    __syncthreads();
  };

  auto theta1 = [&]() {
    const double t = nlock > 0 ? thl[0] : th[0];
    return t > 0 ? t : 1.0;
  };

  // deflate S by the locked columns [n0, n0 + nl) of L (LT holds S L):
  // S <- (I - Ln Ln^T) S (I - Ln Ln^T) = S - Ln W^T - W Ln^T, W = P - Ln (Ln^T P) / 2, P = S Ln
  auto deflate = [&](int n0, int nl) {
    double* Wd = B(iX);  // d x nl (ld nl)
    gram_partial(x, P.L + n0, J, nl, P.LT + n0, J, nl, P.part);
    reduce_bcast(x, P.part, nl * nl, nl, P.red, x.r2s, nl);
    tick(PF_RED);
    for (int r = x.r0 + x.warp; r < x.r1; r += NW)
      for (int c = x.lane; c < nl; c += 32) {
      double s = 0.0;
      for (int l = 0; l < nl; ++l) s = fma(P.L[(int64_t)r * J + n0 + l], x.r2s[l * nl + c], s);
      Wd[(int64_t)r * nl + c] = P.LT[(int64_t)r * J + n0 + c] - 0.5 * s;
    }
    gsync();  // W complete
    // S[own rows][j] -= sum_l Ln[r][l] W[j][l] + W[r][l] Ln[j][l], rows in chunks of 8
    double* lrs = x.r1s;           // [8][nl]
    double* wrs = x.r1s + 8 * nl;  // [8][nl]
    for (int rc = x.r0; rc < x.r1; rc += 8) {
      const int n8 = min(8, x.r1 - rc);
      for (int e = x.tid; e < 8 * nl; e += NT) {
        const int i = e / nl, l = e % nl;
        lrs[e] = i < n8 ? P.L[(int64_t)(rc + i) * J + n0 + l] : 0.0;
        wrs[e] = i < n8 ? Wd[(int64_t)(rc + i) * nl + l] : 0.0;
      }
      __syncthreads();
      for (int j = x.tid; j < d; j += NT) {
        double acc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.0;
        for (int l = 0; l < nl; ++l) {
          const double w = __ldcg(Wd + (int64_t)j * nl + l);
          const double lv = __ldcg(P.L + (int64_t)j * J + n0 + l);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = fma(lrs[i * nl + l], w, fma(wrs[i * nl + l], lv, acc[i]));
        }
        for (int i = 0; i < n8; ++i) S[(int64_t)(rc + i) * d + j] -= acc[i];
      }
      __syncthreads();
    }
  };

  // move the converged leading active vectors into L (prefix, descending order)
  auto lock = [&]() {
    int nl = 0;
    const double th1 = theta1();
    while (nlock + nl < J && nl < ka && rs[nlock + nl] <= P.tol * th1) ++nl;
    if (nl == 0) return;
    if (P.nolock && nlock + nl < J) return;  // debug: lock only when everything converged
    copy_cols(x, B(iQ), ka, P.L + nlock, J, nl);
    copy_cols(x, B(iSQ), ka, P.LT + nlock, J, nl);
    for (int i = x.tid; i < nl; i += NT) thl[nlock + i] = th[nlock + i];
    __syncthreads();
    if (!P.nodefl) deflate(nlock, nl);
    tick(PF_DEFL);
    const int kn = ka - nl;
    // compact Q and SQ into two spare blocks: the new leading dimension makes a
    // CTA's rows overlap other CTAs' old rows, so no block may be rewritten in a
    // new layout before every CTA has finished reading it (grid barrier)
    if (kn > 0) {
      copy_cols(x, B(iQ) + nl, ka, B(iT), kn, kn);
      copy_cols(x, B(iSQ) + nl, ka, B(iY), kn, kn);
      { int t = iQ; iQ = iT; iT = t; }
      { int t = iSQ; iSQ = iY; iY = t; }
    }
    gsync();
    nlock += nl;
    ka = kn;
  };

  // outlier top eigenvalue: power iteration, then lock + deflate it first
  auto power_lock_top = [&]() {
    if (nlock > 0 || ka < 3 || J < 2) return;
    const double t0 = th[0], t1 = th[1];
    if (!(t1 > 0) || t0 < 3.0 * t1) return;
    const double res = rs[0] / t0;
    int npow = (int)ceil(log(fmax(res / P.tol, 1.0)) / -log(t1 / t0)) + 1;
    npow = min(npow, 40);
    double* pq_ = P.pvec[0];
    double* py_ = P.pvec[1];
    copy_cols(x, B(iQ), ka, pq_, 1, 1);
    gsync();
    for (int i = 0; i < npow; ++i) {
      matvec1(x, S, pq_, py_, P.part);
      tick(PF_MV);
      ++matvecs;
      gsync();
      const double nrm = allsum_scalar(x, P.part);
      const double inv = nrm > 0 ? rsqrt(nrm) : 0.0;
      for (int r = x.r0 + x.tid; r < x.r1; r += NT) pq_[r] = py_[r] * inv;
      gsync();
    }
    matvec1(x, S, pq_, py_, P.part);
    tick(PF_MV);
    // theta = q^T y, ||y - theta q||
    {
      __shared__ double w2[NW];
      double s = 0.0;
      for (int r = x.r0 + x.tid; r < x.r1; r += NT) s = fma(pq_[r], py_[r], s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (x.lane == 0) w2[x.warp] = s;
      __syncthreads();
      if (x.tid == 0) {
        double t = 0.0;
        for (int w = 0; w < NW; ++w) t += w2[w];
        P.part[x.G + x.cta] = t;
      }
      __syncthreads();
    }
    gsync();
    const double th0 = allsum_scalar(x, P.part + x.G);
    {
      __shared__ double w3[NW];
      double s = 0.0;
      for (int r = x.r0 + x.tid; r < x.r1; r += NT) {
        const double v = py_[r] - th0 * pq_[r];
        s = fma(v, v, s);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (x.lane == 0) w3[x.warp] = s;
      __syncthreads();
      if (x.tid == 0) {
        double t = 0.0;
        for (int w = 0; w < NW; ++w) t += w3[w];
        P.part[2 * x.G + x.cta] = t;
      }
      __syncthreads();
    }
    gsync();
    const double r0v = sqrt(allsum_scalar(x, P.part + 2 * x.G));
    if (P.dbg && x.cta == 0 && x.tid == 0)
      printf("[eigf] power-lock npow=%d th0=%.9e res=%.3e (tol %.3e)\n", npow, th0, r0v, P.tol * th0);
    if (!(r0v <= P.tol * th0)) return;
    copy_cols(x, pq_, 1, P.L, J, 1);
    copy_cols(x, py_, 1, P.LT, J, 1);
    if (x.tid == 0) {
      thl[0] = th0;
      th[0] = th0;
      rs[0] = r0v;
    }
    __syncthreads();
    deflate(0, 1);
    tick(PF_DEFL);
    const int kn = ka - 1;
    copy_cols(x, B(iQ) + 1, ka, B(iT), kn, kn);
    { int t = iQ; iQ = iT; iT = t; }
    gsync();  // layout change (see lock)
    nlock = 1;
    ka = kn;
    orth_active(2, true);
    rayleigh_ritz();
    lock();
  };

  orth_active(2, true);
  rayleigh_ritz();
  if (P.dbg && x.cta == 0 && x.tid == 0) {
    printf("[eigf] first RR warm=%d\n", P.warm);
    for (int i = 0; i < min(k, 4); ++i) printf("    th[%d]=%.6e res=%.3e\n", i, th[i], rs[i]);
  }
  lock();
  power_lock_top();
  bool converged = nlock >= J || k == d;
  int outer = 0;
  for (; outer < P.max_outer && !converged && !breakdown; ++outer) {
    if (P.dbg && nlock > 0) {
      // diagnostics: |L^T Q|, |S L|, |SQ - S Q|
      gram_partial(x, P.L, J, nlock, B(iQ), ka, ka, P.part);
      reduce_bcast(x, P.part, nlock * ka, ka, P.red, x.r2s, ka);
      double m1 = 0.0;
      for (int e = x.tid; e < nlock * ka; e += NT) m1 = fmax(m1, fabs(x.r2s[e]));
      m1 = gmax(x, m1, P.part);
      gsync();
      matvec(x, S, P.L, J, 1.0, B(iT), 0.0, nullptr, 0.0, nullptr);
      gsync();
      double m2 = 0.0;
      for (int r = x.r0; r < x.r1; ++r)
        for (int c = x.tid; c < nlock; c += NT) m2 = fmax(m2, fabs(B(iT)[(int64_t)r * J + c]));
      m2 = gmax(x, m2, P.part);
      matvec(x, S, B(iQ), ka, 1.0, B(iT), 0.0, nullptr, 0.0, nullptr);
      gsync();
      double m3 = 0.0, m4 = 0.0;
      for (int r = x.r0; r < x.r1; ++r)
        for (int c = x.tid; c < ka; c += NT) {
          m3 = fmax(m3, fabs(B(iT)[(int64_t)r * ka + c] - B(iSQ)[(int64_t)r * ka + c]));
          m4 = fmax(m4, fabs(B(iT)[(int64_t)r * ka + c]));
        }
      m3 = gmax(x, m3, P.part);
      m4 = gmax(x, m4, P.part);
      if (x.cta == 0 && x.tid == 0)
        printf("[eigf-chk] outer=%d nlock=%d ka=%d |L^T Q|=%.3e |S L|=%.3e |SQ - S Q|=%.3e (|S Q|=%.3e)\n", outer,
               nlock, ka, m1, m2, m3, m4);
    }
    const double th1 = theta1();
    const double thJ = th[J - 1];
    const double thtop = th[nlock];
    double b = th[k - 1];
    if (!(b > 0)) b = 1e-12 * th1;
    if (thJ <= b * (1 + 1e-12)) b = thJ * (1 - 1e-3);
    const double a = 0.0;
    const double e = (b - a) / 2, c = (b + a) / 2;
    const double xJ = fmax((thJ - c) / e, 1.0 + 1e-12);
    const double xt = fmax((thtop - c) / e, xJ);
    const double rJ = acosh(xJ), rt = acosh(xt);
    double rmax = 0;
    for (int i = nlock; i < J; ++i) rmax = fmax(rmax, rs[i] / th1);
    int m_need = (int)ceil(log(fmax(rmax / P.tol, 4.0)) / fmax(rJ, 1e-6));
    const int m_amp = max(1, min(16, (int)floor(log(2e7) / fmax(rt, 1e-6))));
    m_need = max(1, min(min(m_need, 64), (m_amp < 6 ? 2 : 8) * m_amp));
    for (int done = 0; done < m_need;) {
      const int mseg = min(m_amp, m_need - done);
      double sigma = e / (thtop - c);
      const double tau = 2.0 / sigma;
      if (done > 0) {
        gsync();
        matvec(x, S, B(iQ), ka, 1.0, B(iSQ), 0.0, nullptr, 0.0, nullptr);
        gsync();
        tick(PF_MV);
        ++matvecs;
      }
      axpby(x, ka, sigma / e, B(iSQ), -c * sigma / e, B(iQ), B(iY));
      int iXp = iQ, iYp = iY;
      int spare[2] = {iX, iT};
      int si = 0;
      for (int i = 2; i <= mseg; ++i) {
        const double sigma2 = 1.0 / (tau - sigma);
        const int iTp = spare[si];
        gsync();
        matvec(x, S, B(iYp), ka, 2 * sigma2 / e, B(iTp), -sigma * sigma2, B(iXp), -2 * sigma2 * c / e,
               B(iYp));
        tick(PF_MV);
        ++matvecs;
        spare[si] = iXp;
        si ^= 1;
        iXp = iYp;
        iYp = iTp;
        sigma = sigma2;
      }
      if (mseg > 1) gsync();  // the filtered block is complete before row-local use
      // the filtered block becomes Q: swap roles so that iQ names it
      if (iYp != iQ) {
        // the five indices stay a permutation: exchange iQ with the holder of the result
        if (iYp == iY) { int t = iQ; iQ = iY; iY = t; }
        else if (iYp == iX) { int t = iQ; iQ = iX; iX = t; }
        else { int t = iQ; iQ = iT; iT = t; }
      }
      done += mseg;
      __syncthreads();
      if (done < m_need) orth_active(1, false);
    }
    orth_active(2, true);
    rayleigh_ritz();
    if (P.dbg && x.cta == 0 && x.tid == 0) {
      printf("[eigf] d=%d J=%d k=%d outer=%d m=%d(amp %d) nlock=%d ka=%d rmax=%.3e th1=%.6e thJ=%.6e thtop=%.6e b=%.6e\n",
             d, J, k, outer, m_need, m_amp, nlock, ka, rmax, th1, thJ, thtop, b);
      for (int i = nlock; i < min(k, nlock + 4); ++i) printf("    th[%d]=%.6e res=%.3e\n", i, th[i], rs[i]);
    }
    __syncthreads();
    lock();
    converged = nlock >= J;
  }

  // outputs: the J leading columns of [L | A], sorted by Ritz value (descending)
  __shared__ int src_of[kMaxBlock + 2];
  {
    const int nc = nlock + ka;
    for (int i = x.tid; i < nc; i += NT) {
      const double v = i < nlock ? thl[i] : th[i];
      int rank = 0;
      for (int q = 0; q < nc; ++q) {
        const double w = q < nlock ? thl[q] : th[q];
        rank += (w > v) || (w == v && q < i);
      }
      src_of[rank] = i;
    }
  }
  __syncthreads();
  {
    for (int r = x.r0 + x.warp; r < x.r1; r += NW)
      for (int j = x.lane; j < J; j += 32) {
      const int s = src_of[j];
      P.outV[(int64_t)r * J + j] = s < nlock ? P.L[(int64_t)r * J + s] : B(iQ)[(int64_t)r * ka + (s - nlock)];
    }
    // warm-start basis [L | A]
    for (int r = x.r0 + x.warp; r < x.r1; r += NW)
      for (int c = x.lane; c < k; c += 32) {
      P.basis[(int64_t)r * k + c] = c < nlock ? P.L[(int64_t)r * J + c] : B(iQ)[(int64_t)r * ka + (c - nlock)];
    }
  }
  if (x.cta == 0) {
    for (int j = x.tid; j < J; j += NT) {
      const int s = src_of[j];
      P.theta_out[j] = s < nlock ? thl[s] : th[s];
    }
    if (x.tid < 8) P.prof[x.tid] += pacc[x.tid];
    if (x.tid == 0) {
      P.info[0] = converged ? 1 : 0;
      P.info[1] = outer;
      P.info[2] = matvecs;
      P.info[3] = jsw;
      P.info[4] = breakdown;
    }
  }
}

// Unit-test kernel for the tiled product: Out = alpha S Y + gamma D (all CTAs).
__global__ void __launch_bounds__(NT, 1) k_eigf_unit_mv(const double* S, const double* Y, int d, int n,
                                                       double alpha, double* Out, double gamma,
                                                       const double* D, int reps) {
  extern __shared__ __align__(16) double smem[];
  Ctx x;
  x.cta = blockIdx.x;
  x.G = gridDim.x;
  x.tid = threadIdx.x;
  x.warp = x.tid >> 5;
  x.lane = x.tid & 31;
  x.d = d;
  x.r0 = x.r1 = 0;
  x.r1s = smem;
  x.r2s = smem;
  for (int i = 0; i < reps; ++i) matvec(x, S, Y, n, alpha, Out, gamma, D, 0.0, nullptr);
}

// Unit-test kernel for the k x k device routines (one CTA): mode 0 -> CholQR
// factor M of SPD `in` (out = M, k x k); mode 1 -> Jacobi (out = V with
// eigenvectors in columns, theta = eigenvalues descending, iout[0] = sweeps).
__global__ void __launch_bounds__(NT, 1) k_eigf_unit(int mode, const double* in, int k, double* out,
                                                    double* theta, int* iout, int sweeps, double shift) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double th[kMaxBlock + 2];
  __shared__ int perm[kMaxBlock + 2];
  Ctx x;
  x.cta = 0;
  x.G = 1;
  x.tid = threadIdx.x;
  x.warp = x.tid >> 5;
  x.lane = x.tid & 31;
  x.d = k;
  x.r0 = 0;
  x.r1 = k;
  const int kp = k + (k & 1), ld = kp + 1;
  x.r1s = smem;
  x.r2s = smem + (size_t)kp * ld;
  for (int r = x.warp; r < k; r += NW)
    for (int c = x.lane; c < k; c += 32) x.r1s[r * ld + c] = in[r * k + c];
  __syncthreads();
  if (mode == 0) {
    cholqr_factor(x, x.r1s, x.r2s, k, ld, shift);
    for (int r = x.warp; r < k; r += NW)
      for (int c = x.lane; c < k; c += 32) out[r * k + c] = x.r2s[r * ld + c];
  } else {
    const int sw = jacobi(x, x.r1s, x.r2s, k, sweeps, 1e-13, th, perm);
    for (int r = x.warp; r < k; r += NW)
      for (int c = x.lane; c < k; c += 32) out[r * k + c] = x.r2s[perm[c] * ld + r];
    for (int i = x.tid; i < k; i += NT) theta[i] = th[i];
    if (x.tid == 0) iout[0] = sw;
  }
}

}  // namespace

size_t eig_fused_smem(int k, int d, int G) {
  const int kp = k + (k & 1);
  const int R = (int)((d + G - 1) / G);
  const size_t jac = (region1_doubles(kp, R) + (size_t)kp * (kp + 1)) * sizeof(double);
  // product: the largest plan over the active widths n <= k
  size_t mv = 0;
  for (int n = 1; n <= k; ++n) {
    const MvPlan pl = mv_plan(d, n, G);
    const int ng = (pl.tpb + 1) / 2, KS = NW / ng;
    const size_t st = mv_smem_doubles(pl.m8, pl.tpb);
    const size_t ep = (size_t)KS * 8 * pl.m8 * 8 * pl.tpb;
    mv = std::max(mv, std::max(st, ep) * sizeof(double));
  }
  const size_t gp = (size_t)R * 2 * kp * sizeof(double);
  return std::max(jac, std::max(mv, gp));
}

bool eig_fused(double* S, int64_t d, int J, EigSlot& slot, EigWs& ws, const EigOpts& o, double* out_V,
               double* theta_dev, int* info_dev, cudaStream_t st) {
  static int nsm = 0;
  static size_t smem_set = 0;
  int k = J + (o.oversample > 0 ? o.oversample : std::max(8, std::min(J, 32)));
  if (k > kMaxBlock) k = kMaxBlock;
  if (k > d) k = (int)d;
  if (k & 1) k = (k + 1 <= kMaxBlock && k + 1 <= d) ? k + 1 : k - 1;
  if (k < J) k = J;
  if (nsm == 0) {
    int dev = 0;
    TK_CUDA(cudaGetDevice(&dev));
    TK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  }
  const int grid = nsm;  // one CTA per SM (cooperative: all co-resident)
  const size_t smem = eig_fused_smem(k, (int)d, grid);
  if (smem + 8 * 1024 > 227 * 1024) fail(TUCKER_E_ARG, "eig_fused: block too large for shared memory");
  if (smem > smem_set) {
    TK_CUDA(cudaFuncSetAttribute(k_eig_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    smem_set = smem;
  }
  {
    int per = 0;
    TK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_eig_fused, NT, smem));
    if (per < 1) fail(TUCKER_E_CUDA, "eig_fused: kernel cannot be resident");
  }
  const size_t dk = (size_t)d * k;
  ws.Q.ensure(dk);
  ws.SQ.ensure(dk);
  ws.X.ensure(dk);
  ws.Y.ensure(dk);
  ws.T.ensure(dk);
  ws.L.ensure((size_t)d * J);
  ws.LT.ensure((size_t)d * J);
  ws.fpart.ensure((size_t)grid * std::max<size_t>((size_t)k * k, 3));
  ws.fred.ensure((size_t)k * k);
  ws.pq.ensure((size_t)d);
  ws.py.ensure((size_t)d);
  slot.basis.ensure(dk);
  FusedArgs a;
  a.S = S;
  a.d = (int)d;
  a.J = J;
  a.k = k;
  a.blk[0] = ws.Q.p;
  a.blk[1] = ws.SQ.p;
  a.blk[2] = ws.X.p;
  a.blk[3] = ws.Y.p;
  a.blk[4] = ws.T.p;
  a.L = ws.L.p;
  a.LT = ws.LT.p;
  a.part = ws.fpart.p;
  a.red = ws.fred.p;
  a.pvec[0] = ws.pq.p;
  a.pvec[1] = ws.py.p;
  a.basis = slot.basis.p;
  a.warm = (slot.valid && slot.d == d && slot.k == k) ? 1 : 0;
  a.outV = out_V;
  a.theta_out = theta_dev;
  a.info = info_dev;
  ws.fprof.ensure(8);
  if (!ws.fprof_init) {
    TK_CUDA(cudaMemsetAsync(ws.fprof.p, 0, 8 * sizeof(long long), st));
    ws.fprof_init = true;
  }
  a.prof = ws.fprof.p;
  a.tol = o.tol;
  a.max_outer = o.max_outer;
  a.jsweeps = o.jacobi_sweeps;
  a.seed = 0x5eed0000ull + (uint64_t)d * 131 + (uint64_t)J;
  static const bool dbg = std::getenv("TUCKER_EIG_DEBUG") != nullptr;
  a.dbg = dbg ? 1 : 0;
  {
    const char* e = std::getenv("TUCKER_EIG_JSW");
    if (e) a.jsweeps = std::atoi(e);
    a.noshift = std::getenv("TUCKER_EIG_NOSHIFT") != nullptr;
    a.nolock = std::getenv("TUCKER_EIG_NOLOCK") != nullptr;
    a.nodefl = std::getenv("TUCKER_EIG_NODEFL") != nullptr;
  }
  void* args[] = {&a};
  TK_CUDA(cudaLaunchCooperativeKernel((const void*)k_eig_fused, dim3(grid), dim3(NT), args, smem, st));
  if (g_launch_counter) ++(*g_launch_counter);
  if (sync_check_enabled()) TK_CUDA(cudaStreamSynchronize(st));
  slot.d = d;
  slot.k = k;
  slot.valid = true;
  return true;
}

void eig_unit_mv(const double* S, const double* Y, int d, int n, double alpha, double* Out, double gamma,
                 const double* D, cudaStream_t st) {
  int nsm = 0, dev = 0;
  TK_CUDA(cudaGetDevice(&dev));
  TK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  size_t mv = 0;
  for (int nn = 1; nn <= n; ++nn) {
    const MvPlan pl = mv_plan(d, nn, nsm);
    const int ng = (pl.tpb + 1) / 2, KS = NW / ng;
    mv = std::max(mv, std::max(mv_smem_doubles(pl.m8, pl.tpb), (size_t)KS * 64 * pl.m8 * pl.tpb));
  }
  const size_t smem = mv * sizeof(double);
  TK_CUDA(cudaFuncSetAttribute(k_eigf_unit_mv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  TK_LAUNCH(k_eigf_unit_mv, nsm, NT, smem, st, S, Y, d, n, alpha, Out, gamma, D, 1);
}

double eig_unit_mv_time(int d, int n, int reps) {
  DBuf<double> S((size_t)d * d), Y((size_t)d * n), O((size_t)d * n);
  TK_CUDA(cudaMemset(S.p, 0, S.bytes()));
  TK_CUDA(cudaMemset(Y.p, 0, Y.bytes()));
  eig_unit_mv(S.p, Y.p, d, n, 1.0, O.p, 0.0, nullptr, 0);  // sets the smem attribute
  int nsm = 0, dev = 0;
  TK_CUDA(cudaGetDevice(&dev));
  TK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  size_t mv = 0;
  for (int nn = 1; nn <= n; ++nn) {
    const MvPlan pl = mv_plan(d, nn, nsm);
    const int ng = (pl.tpb + 1) / 2, KS = NW / ng;
    mv = std::max(mv, std::max(mv_smem_doubles(pl.m8, pl.tpb), (size_t)KS * 64 * pl.m8 * pl.tpb));
  }
  const size_t smem = mv * sizeof(double);
  cudaEvent_t a, b;
  TK_CUDA(cudaEventCreate(&a));
  TK_CUDA(cudaEventCreate(&b));
  // (T(1 + reps) - T(1)) / reps: one launch, products after the first reuse the plan
  float ms1 = 0, ms2 = 0;
  TK_CUDA(cudaEventRecord(a, 0));
  k_eigf_unit_mv<<<nsm, NT, smem, 0>>>(S.p, Y.p, d, n, 1.0, O.p, 0.0, nullptr, 1);
  TK_CUDA(cudaEventRecord(b, 0));
  TK_CUDA(cudaEventSynchronize(b));
  TK_CUDA(cudaEventElapsedTime(&ms1, a, b));
  TK_CUDA(cudaEventRecord(a, 0));
  k_eigf_unit_mv<<<nsm, NT, smem, 0>>>(S.p, Y.p, d, n, 1.0, O.p, 0.0, nullptr, 1 + reps);
  TK_CUDA(cudaEventRecord(b, 0));
  TK_CUDA(cudaEventSynchronize(b));
  TK_CUDA(cudaEventElapsedTime(&ms2, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return 1e3 * (ms2 - ms1) / reps;
}

void eig_unit(int mode, const double* in, int k, double* out, double* theta, int* iout, int sweeps,
              double shift, cudaStream_t st) {
  const int kp = k + (k & 1);
  const size_t smem = (size_t)2 * kp * (kp + 1) * sizeof(double);
  TK_CUDA(cudaFuncSetAttribute(k_eigf_unit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  TK_LAUNCH(k_eigf_unit, 1, NT, smem, st, mode, in, k, out, theta, iout, sweeps, shift);
}

}  // namespace tk
