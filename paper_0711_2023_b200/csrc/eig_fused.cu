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
//   * S * Y: 2D tiles on the fp64 tensor cores (DMMA), operands streamed by TMA
//     bulk copies; a barrier follows every product (it is not row-local).
//   * k x k reductions (Q^T Q, Q^T S Q, Ritz residuals): per-CTA partials over
//     its rows, a distributed fixed-order sum (deterministic), then every CTA
//     loads the result and runs the small dense step (LDL^T-based CholQR
//     factor, Jacobi) REDUNDANTLY in its own shared memory -- no further
//     barrier, and the k x k result is where the row-local apply needs it.
//
// Layout (eig_layout): S is LS x LS-strided with RP rows, LS = round_up(d, 64),
// RP = LS + 64; the d x k work blocks have leading dimension LB = k rounded up
// to even and RP rows.  Everything outside the d x d / d x k data is zero, so
// the product streams whole 64-wide K chunks and whole row tiles with no edge
// cases, and every bulk copy is 16-byte aligned.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace tk {
namespace {

constexpr int NT = 512;  // threads per CTA
constexpr int NW = NT / 32;

struct FusedArgs {
  double* S;   // RP x LS (deflated in place; padding zeroed by the kernel)
  int d, J, k;
  int ls, lb, rp;           // S stride, block stride, padded rows
  int mv_m8, mv_rb, mv_kb, mv_kc;  // product plan (FusedArgs)
  int sres_off;             // offset (doubles) of the resident S tile in dynamic smem, -1: streamed
  double* blk[5];           // five RP x LB work blocks (roles rotate)
  double* L;                // d x J locked vectors
  double* LT;               // d x J  S L
  double* part;             // [G][k*k] reduction partials
  double* red;              // [k*k] reduced result
  double* pvec[3];          // power iteration / Lanczos vectors (d)
  double* mpart;            // [KB][RPX][LB] split-K partial products
  double* basis;            // d x LB warm-start basis (read if warm, always written)
  int warm;
  int warm_exact;           // basis = the slot's previous [L | Q] (orthonormal): no initial CholQR
  double* outV;             // d x J output (ld = J)
  double* theta_out;        // J
  long long* prof;          // [8] per-phase ns (CTA 0's view), accumulated; [8] algorithmic flops
  int* info;                // [0] converged [1] outer [2] matvecs [3] jacobi sweeps [4] breakdown
  double* dinfo;            // [0] lambda_min estimate (0: not estimated) [1] last filter bound b
  int lanczos;              // estimate lambda_min (Lanczos) for the filter's lower bound
  double lmin_hint;         // else: lower bound carried over from the slot's last solve (0: none)
  double tol;
  int max_outer, jsweeps, jsweeps0;
  uint64_t seed;
  int dbg;
};

// region 1 holds a k x (k+1) matrix or the own-row staging of a d x k block
__host__ __device__ inline size_t region1_doubles(int kp, int R) {
  const size_t a = (size_t)kp * (kp + 1), b = (size_t)R * kp;
  return a > b ? a : b;
}

struct Ctx {
  int cta, G, tid, warp, lane;
  int d, r0, r1;  // own rows [r0, r1)
  int ls, lb;     // S stride, block stride
  int mv_m8, mv_rb, mv_kb, mv_kc;  // product plan (mv_plan(d, G)), computed on the host
  double* r1s;    // smem region 1 (k x (k+1) doubles or staging)
  double* r2s;    // smem region 2 (k x (k+1) doubles)
  double* sres;   // resident S tile of the product plan (nullptr: S is streamed)
};

// TK_GSYNC_STATS=1 (debug builds): count grid barriers and their time as seen
// by CTA 0 (the timer reads delay CTA 0's arrival, so it is off by default)
#ifndef TK_GSYNC_STATS
#define TK_GSYNC_STATS 0
#endif
// TK_EIG_PROFILE=1 (profiling builds, TUCKER_NVCC_EXTRA): per-phase and
// per-product globaltimer accounting by CTA 0 (tucker_stats eig_phase_ms /
// product_ms).  Off by default: the timer reads sit on CTA 0's path into the
// next grid barrier, which every CTA waits for.
#ifndef TK_EIG_PROFILE
#define TK_EIG_PROFILE 0
#endif
__device__ unsigned long long g_gsync_stat[2];  // [0] barriers, [1] ns (CTA 0's view; debug)
__device__ __forceinline__ void gsync() {
#if TK_GSYNC_STATS
  long long t0 = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#endif
  cg::this_grid().sync();
#if TK_GSYNC_STATS
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    g_gsync_stat[0] += 1;
    g_gsync_stat[1] += (unsigned long long)(t1 - t0);
  }
#endif
}

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

// deterministic uniform(-1, 1) fill of the own rows of Q (k columns, stride ld)
__device__ void fill_random(const Ctx& x, double* Q, int ld, int k, uint64_t seed) {
  for (int r = x.r0 + x.warp; r < x.r1; r += NW)
    for (int c = x.lane; c < k; c += 32) {
      const uint64_t h = mix64(seed ^ mix64((uint64_t)r * 1315423911ull + (uint64_t)c));
      Q[(int64_t)r * ld + c] = ((double)(h >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
    }
}

// z = a x + b y on own rows (n columns, stride ld), z may alias x or y
__device__ void axpby(const Ctx& x, int n, int ld, double a, const double* X, double b, const double* Y,
                      double* Z) {
  for (int r = x.r0 + x.warp; r < x.r1; r += NW)
    for (int c = x.lane; c < n; c += 32) {
      const int64_t o = (int64_t)r * ld + c;
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

// zero the padding of S (columns [d, LS) of rows < d, rows [d, RP)) and the
// padding rows [d, RP) of the work blocks, distributed over the CTAs
__device__ void zero_padding(const Ctx& x, double* S, int rp, double* const* blk) {
  for (int r = x.r0 + x.warp; r < x.r1; r += NW)
    for (int c = x.d + x.lane; c < x.ls; c += 32) S[(int64_t)r * x.ls + c] = 0.0;
  for (int r = x.d + x.cta; r < rp; r += x.G) {
    for (int c = x.tid; c < x.ls; c += NT) S[(int64_t)r * x.ls + c] = 0.0;
    for (int b = 0; b < 5; ++b)
      for (int c = x.tid; c < x.lb; c += NT) blk[b][(int64_t)r * x.lb + c] = 0.0;
  }
}

// ------------------------------------------------- S * Y on the fp64 tensor cores --
constexpr int KCH = 64;          // padding granule of the layout (K chunks stay whole)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ------------------------------------------------- S * Y on the fp64 tensor cores --
// Split-K plan: row blocks of MT rows (MT = 8 m8, m8 <= 8) x K ranges of kchunk
// (multiple of 64) with RB * KB <= G CTAs, minimising the per-CTA work MT kchunk
// (ties: larger MT, less partial traffic).  Depends on d only.
struct MvPlan {
  int m8, RB, KB, kchunk;
};
__host__ __device__ inline MvPlan mv_plan(int d, int G) {
  const int LS = (d + 63) / 64 * 64;
  // d > 64 G (e.g. MP's d = 50000 at config 5): 64-row blocks over the full K range,
  // more blocks than CTAs -- every CTA loops over its blocks (matvec)
  MvPlan best{8, (d + 63) / 64, 1, LS};
  long long bc = -1;
  for (int m8 = 8; m8 >= 1; --m8) {
    const int MT = 8 * m8;
    const int RB = (d + MT - 1) / MT;
    const int kbmax = G / RB;
    if (kbmax < 1) continue;
    const int kc = ((LS + kbmax - 1) / kbmax + 63) / 64 * 64;
    const int KB = (LS + kc - 1) / kc;
    const long long cost = (long long)MT * kc;
    if (bc < 0 || cost < bc) {
      bc = cost;
      best = MvPlan{m8, RB, KB, kc};
    }
  }
  return best;
}
constexpr int KC2 = 64;  // K per staged chunk inside a CTA's range
__host__ __device__ inline int mv_ypad(int n8) { return ((8 * n8 + 15) & ~15) + 4; }  // = 4 or 12 mod 16
__host__ __device__ inline size_t mv_stage_doubles(int m8, int n8) {
  const int Mg = (m8 + 1) / 2, Ng = NW / Mg, GN = (n8 + Ng - 1) / Ng;
  return (size_t)16 * Mg * (KC2 + 4) + (size_t)KC2 * mv_ypad(GN * Ng);
}
__host__ __device__ inline size_t mv_smem_doubles(int m8, int n8) { return 2 * mv_stage_doubles(m8, n8); }

// Out = alpha S Y + gamma D + delta E on the padded layout (S RP x LS, Y/Out/D/E
// RP x LB, n <= 116 active columns).  Phase A (every CTA (rb, kb) of the plan):
// partial P_kb[rows of rb][0..8 n8) = S[rows, K range] Y[K range, :] on DMMA,
// K streamed in 64-wide chunks through a double-buffered 16-byte cp.async ring;
// warp w owns m-tile pair (w / Ng) x n-tile group (w mod Ng) (<= 2 x 4
// accumulator tiles).  Partials go to `mpart` ([KB][RP][LB]).  Barrier.  Phase B
// (row owners, row-local): Out = alpha sum_kb P_kb + gamma D + delta E in a
// fixed order.  Y, D, E must be complete before the call (barrier); Out may
// alias D or E (each element is read before it is written by the same thread).
// Phase A of the product for one CTA tile, every warp on a uniform 2 x GN block
// of 8x8 DMMA tiles (m-tile pair mg x n-tile group ng; tiles beyond the CTA's
// rows / the active columns are computed on padding and not stored), so the
// inner loop is straight-line code with no per-tile predicates.
struct PhaseA {
  const double* S;     // global S (row stride LS), used when the tile is streamed
  const double* Y;     // global Y (row stride LB)
  double* P;           // partial product of this K range (row stride LB)
  double* stage;       // shared staging (2 buffers)
  const double* sres;  // resident S tile (row stride SPR) or nullptr
  int LS, LB, n, MT, MT2, row0, kbeg, nch, SPR, YP, Ng, Mg, tid, warp, lane;
};

template <int GN>
__device__ __noinline__ void mv_phase_a(const PhaseA a) {
  constexpr int SPK = KC2 + 4;
  const int YC = 8 * GN * a.Ng;  // staged Y columns
  const size_t STG = (size_t)a.MT2 * SPK + (size_t)KC2 * a.YP;
  const int mg = a.warp / a.Ng, ng = a.warp - mg * a.Ng;
  const bool wact = mg < a.Mg;
  const int mt0 = 2 * mg, nt0 = ng * GN;
  const bool res = a.sres != nullptr;
  const double* gS = a.S + (int64_t)a.row0 * a.LS;
  auto stage = [&](int buf, int k0) {
    double* sS = a.stage + (size_t)buf * STG;
    double* sY = sS + a.MT2 * SPK;
    if (!res)
      for (int u = a.tid; u < a.MT2 * (KC2 / 2); u += NT) {
        const int r = u >> 5, c2 = (u & 31) << 1;
        cp_async16(sS + r * SPK + c2, gS + (int64_t)r * a.LS + k0 + c2);
      }
    const int yu = YC >> 1;
    for (int kk = a.warp; kk < KC2; kk += NW) {
      const double* src = a.Y + (int64_t)(k0 + kk) * a.LB;
      double* dst = sY + kk * a.YP;
      for (int u = a.lane; u < yu; u += 32) cp_async16(dst + 2 * u, src + 2 * u);
    }
    cp_commit();
  };
  double acc[2][GN][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < GN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int ar = a.lane >> 2, aq = a.lane & 3;
  stage(0, a.kbeg);
  for (int ch = 0; ch < a.nch; ++ch) {
    if (ch + 1 < a.nch) {
      stage((ch + 1) & 1, a.kbeg + (ch + 1) * KC2);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (wact) {
      const double* sS = a.stage + (size_t)(ch & 1) * STG;
      const double* sY = sS + a.MT2 * SPK;
      const double* aS = res ? a.sres + ch * KC2 : sS;
      const int aLD = res ? a.SPR : SPK;
      const double* ap0 = aS + (8 * mt0 + ar) * aLD + aq;
      const double* ap1 = ap0 + 8 * aLD;
      const double* bp = sY + aq * a.YP + 8 * nt0 + ar;
      const int bstep = 4 * a.YP;
#pragma unroll 4
      for (int kb4 = 0; kb4 < KC2; kb4 += 4) {
        const double a0 = ap0[kb4], a1 = ap1[kb4];
        double b[GN];
#pragma unroll
        for (int j = 0; j < GN; ++j) b[j] = bp[8 * j];
        bp += bstep;
#pragma unroll
        for (int j = 0; j < GN; ++j) {
          dmma(acc[0][j][0], acc[0][j][1], a0, b[j]);
          dmma(acc[1][j][0], acc[1][j][1], a1, b[j]);
        }
      }
    }
    __syncthreads();  // buffer (ch & 1) free for chunk ch + 2
  }
  if (wact) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < GN; ++j) {
        const int rl = 8 * (mt0 + i) + ar, c = 8 * (nt0 + j) + 2 * aq;
        if (rl < a.MT) {
          double* pr = a.P + (int64_t)(a.row0 + rl) * a.LB;
          if (c < a.n) pr[c] = acc[i][j][0];
          if (c + 1 < a.n) pr[c + 1] = acc[i][j][1];
        }
      }
  }
}

// Out = alpha S Y + gamma D + delta E on the padded layout (S RP x LS, Y/Out/D/E
// RP x LB, n <= 116 active columns).  Phase A (every CTA (rb, kb) of the plan):
// partial P_kb[rows of rb][0..n) = S[rows, K range] Y[K range, :] on DMMA
// (mv_phase_a), K streamed in 64-wide chunks through a double-buffered 16-byte
// cp.async ring (S from the resident tile when it fits in shared memory).
// Partials go to `mpart` ([KB][RPX][LB]).  Barrier.  Phase B (row owners,
// row-local): Out = alpha sum_kb P_kb + gamma D + delta E in a fixed order.
// Y, D, E must be complete before the call (barrier); Out may alias D or E
// (each element is read before it is written by the same thread).
__device__ void matvec(const Ctx& x, double* mpart, const double* S, const double* Y, int n, double alpha,
                       double* Out, double gamma, const double* Dm, double delta, const double* Em,
                       long long* mvt = nullptr) {
  long long t0 = mvt ? gtimer() : 0;
  const MvPlan pl{x.mv_m8, x.mv_rb, x.mv_kb, x.mv_kc};
  const int LS = x.ls, LB = x.lb;
  const int n8 = (n + 7) >> 3;
  const int RPX = (x.d + 8 * pl.m8 - 1) / (8 * pl.m8) * (8 * pl.m8);  // rows covered by the plan
  for (int t = x.cta; t < pl.RB * pl.KB; t += x.G) {  // one pass unless the plan has more blocks than CTAs
    const int rb = t / pl.KB, kb = t - rb * pl.KB;
    PhaseA a;
    a.S = S;
    a.Y = Y;
    a.P = mpart + (size_t)kb * RPX * LB;
    a.stage = x.r1s;
    a.sres = x.sres;
    a.LS = LS;
    a.LB = LB;
    a.n = n;
    a.MT = 8 * pl.m8;
    a.Mg = (pl.m8 + 1) >> 1;
    a.MT2 = 16 * a.Mg;
    a.row0 = rb * a.MT;
    a.kbeg = kb * pl.kchunk;
    a.nch = (min(LS, a.kbeg + pl.kchunk) - a.kbeg) / KC2;
    a.SPR = pl.kchunk + 4;
    a.Ng = NW / a.Mg;
    const int GN = (n8 + a.Ng - 1) / a.Ng;  // 1..4
    a.YP = mv_ypad(GN * a.Ng);
    a.tid = x.tid;
    a.warp = x.warp;
    a.lane = x.lane;
    switch (GN) {
      case 1: mv_phase_a<1>(a); break;
      case 2: mv_phase_a<2>(a); break;
      case 3: mv_phase_a<3>(a); break;
      default: mv_phase_a<4>(a); break;
    }
  }
  long long t1 = mvt ? gtimer() : 0;
  gsync();
  long long t2 = mvt ? gtimer() : 0;
  // phase B: own rows; the (row, column) items are spread over all threads
  // (a CTA owns ~d/G rows, fewer than its warps) with 8 partial loads in flight
  const int nrow = x.r1 - x.r0;
  const size_t pstr = (size_t)RPX * LB;
  for (int it = x.tid; it < nrow * n; it += NT) {
    const int rr = it / n, c = it - rr * n;
    const int r = x.r0 + rr;
    const double* pp0 = mpart + (size_t)r * LB + c;
    const int64_t o = (int64_t)r * LB + c;
    const double dv = gamma != 0.0 ? Dm[o] : 0.0, ev = delta != 0.0 ? Em[o] : 0.0;
    double sum = 0.0;
    int q = 0;
    for (; q + 8 <= pl.KB; q += 8) {  // summed in order
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(pp0 + (q + u) * pstr);
#pragma unroll
      for (int u = 0; u < 8; ++u) sum += v[u];
    }
    for (; q < pl.KB; ++q) sum += __ldcg(pp0 + q * pstr);
    double val = alpha * sum;
    if (gamma != 0.0) val += gamma * dv;
    if (delta != 0.0) val += delta * ev;
    Out[o] = val;
  }
  __syncthreads();  // own rows of Out complete for any thread mapping
  if (mvt) {
    const long long t3 = gtimer();
    mvt[0] += t1 - t0;
    mvt[1] += t2 - t1;
    mvt[2] += t3 - t2;
  }
}

// (re)load this CTA's tile of S for the product plan into x.sres (after a barrier
// that makes S complete); rows [rb MT, +MT) x K range [kb kchunk, +kchunk)
__device__ void load_sres(const Ctx& x, const double* S) {
  if (!x.sres || x.cta >= x.mv_rb * x.mv_kb) return;
  const int rb = x.cta / x.mv_kb, kb = x.cta - rb * x.mv_kb;
  const int MT = 8 * x.mv_m8, MT2 = 16 * ((x.mv_m8 + 1) / 2), SPR = x.mv_kc + 4;
  const int kbeg = kb * x.mv_kc, klen = min(x.ls - kbeg, x.mv_kc);
  const double* g = S + (int64_t)rb * MT * x.ls + kbeg;
  const int upr = klen >> 1;  // 16-byte units per row
  for (int u = x.tid; u < MT2 * upr; u += NT) {  // MT2 >= MT rows (padding rows are never stored)
    const int r = u / upr, c2 = (u - r * upr) << 1;
    cp_async16(x.sres + r * SPR + c2, g + (int64_t)r * x.ls + c2);
  }
  cp_commit();
  cp_wait<0>();
  __syncthreads();
}

// single vector: y[own rows] = S[own rows, :] q, partial ||y||^2 -> part[cta]
__device__ void matvec1(const Ctx& x, const double* S, const double* q, double* y, double* part) {
  __shared__ double wsum[NW];
  double nrm = 0.0;
  for (int r = x.r0 + x.warp; r < x.r1; r += NW) {
    const double* srow = S + (int64_t)r * x.ls;
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

// partial over own rows of a per-row scalar -> part[cta] (block sum, fixed order)
__device__ void block_partial(const Ctx& x, double v, double* part) {
  __shared__ double w2[NW];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (x.lane == 0) w2[x.warp] = v;
  __syncthreads();
  if (x.tid == 0) {
    double t = 0.0;
    for (int w = 0; w < NW; ++w) t += w2[w];
    part[x.cta] = t;
  }
  __syncthreads();
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
// part[i*nb + j][cta] = sum_{own rows r} A[r][i] B[r][j]
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
  // entry-major partials: part[e * G + cta] (reduce_bcast reads each entry's G
  // partials as one contiguous run)
  for (int i = x.warp; i < na; i += NW)
    for (int j = x.lane; j < nb; j += 32) {
      double s = 0.0;
      for (int r = 0; r < nr; ++r) s = fma(sA[r * na + i], sB[r * nb + j], s);
      part[(size_t)(i * nb + j) * x.G + x.cta] = s;
    }
  __syncthreads();
}

// red[e] = sum_z part[e][z] (entry-major partials, fixed order), entries distributed over CTAs; then
// barrier and every CTA copies red into dst (smem, row stride ldd, nb columns).
// Loads are issued in batches (independent registers) so each phase costs about
// one L2 round trip instead of one per element.
__device__ void reduce_bcast(const Ctx& x, const double* part, int E, int nb, double* red, double* dst,
                             int ldd) {
  gsync();
  const int per = (E + x.G - 1) / x.G;
  const int e0 = x.cta * per, e1 = min(E, e0 + per);
  // tpe threads per entry (the largest power of two <= 32 that keeps the CTA's
  // entries in one pass), each a strided subset of the partials with 8 loads in
  // flight, combined by shuffles in a fixed pattern (depends on E and G only:
  // deterministic)
  int tpe = 32;
  while (tpe > 1 && tpe * per > NT) tpe >>= 1;
  for (int base = e0; base < e1; base += NT / tpe) {
    const int e = base + x.tid / tpe, sub = x.tid % tpe;
    double s = 0.0;
    if (e < e1) {
      for (int z0 = sub; z0 < x.G; z0 += 8 * tpe) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int z = z0 + u * tpe;
          v[u] = z < x.G ? __ldcg(part + (size_t)e * x.G + z) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
      }
    }
    for (int o = 1; o < tpe; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (e < e1 && sub == 0) red[e] = s;
  }
  gsync();
  const int nrow = E / nb;
  constexpr int B8 = 8;
  for (int e0b = 0; e0b < E; e0b += NT * B8) {
    double v[B8];
#pragma unroll
    for (int t = 0; t < B8; ++t) {
      const int e = e0b + x.tid + NT * t;
      v[t] = e < E ? __ldcg(red + e) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < B8; ++t) {
      const int e = e0b + x.tid + NT * t;
      if (e < E) {
        const int i = e / nb;
        dst[i * ldd + (e - i * nb)] = v[t];
      }
    }
  }
  (void)nrow;
  __syncthreads();
}

// fp64 reciprocal / reciprocal square root from the hardware approximations plus
// Newton steps -- short dependency chains instead of the IEEE division / sqrt
// sequences.
__device__ __forceinline__ double rcp_nt(double x) {
  double r = (double)__frcp_rn((float)x);
  r = r * fma(-x, r, 2.0);
  r = r * fma(-x, r, 2.0);
  return r;
}
__device__ __forceinline__ double rsqrt_nt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

// ---------------------------------------------------------- CholQR factor --
// G (k x k, in A = smem, ld) SPD.  Equilibrate (D G D + shift I, D = diag^-1/2)
// and eliminate symmetrically on [A | E] (E = I): after step j rows l > j of
// the upper part are reduced and E accumulates L^{-1} (G = L P L^T, P the
// pivots).  Then M = D E^T P^{-1/2} (upper triangular) satisfies M^T G M = I,
// written to X (smem, ld): Q M has orthonormal columns (CholQR).  One barrier
// per elimination step.
// 1/x from the fp64 reciprocal approximation plus two Newton steps (x > 0
// normal): a short dependency chain on the elimination's critical path
__device__ __forceinline__ double rcp_nt64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-x, r, 2.0);
  r = r * fma(-x, r, 2.0);
  return r;
}
__device__ void cholqr_factor(const Ctx& x, double* A, double* X, int k, int ld, double shift) {
  __shared__ double dsc[kMaxBlock];
  __shared__ double piv[kMaxBlock];
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
  // Two elimination steps (pivots j, j+1) per barrier: row l > j+1 applies step
  // j and, with row j+1's step-j values formed on the fly, step j+1.  Row j+1
  // itself (its E part and its pivot) is brought up to date in the NEXT period,
  // when no row reads it any more.
  int jd = -1;  // row whose update is deferred (-1: none): E[jd] -= fd E[jd-1], A[jd][jd] = pd
  double fd = 0.0, pd = 0.0;
  int j = 0;
  for (; j + 2 < k; j += 2) {
    const double a00 = A[j * ld + j], a01 = A[j * ld + j + 1], a11 = A[(j + 1) * ld + j + 1];
    const double ip0 = rcp_nt64(a00 > 1e-12 ? a00 : 1e-12);
    const double f1 = a01 * ip0;
    const double p1 = fma(-f1, a01, a11);
    const double ip1 = rcp_nt64(p1 > 1e-12 ? p1 : 1e-12);
    if (jd >= 0 && x.warp == NW - 1) {  // deferred: row jd (= previous j + 1)
      double* el = X + jd * ld;
      const double* ej = X + (jd - 1) * ld;
      for (int m = x.lane; m < jd; m += 32) el[m] = fma(-fd, ej[m], el[m]);
      if (x.lane == 0) A[jd * ld + jd] = pd;
    }
    const double* aj = A + j * ld;
    const double* aj1 = A + (j + 1) * ld;
    const double* ej = X + j * ld;
    const double* ej1 = X + (j + 1) * ld;
    for (int l = j + 2 + x.warp; l < k; l += NW) {
      const double f = aj[l] * ip0;
      const double g = fma(-f1, aj[l], aj1[l]) * ip1;  // A'[j+1][l] / p1
      double* al = A + l * ld;
      for (int m = l + x.lane; m < k; m += 32) {
        const double u = aj[m];
        al[m] = fma(-g, fma(-f1, u, aj1[m]), fma(-f, u, al[m]));
      }
      double* el = X + l * ld;
      for (int m = x.lane; m <= j + 1; m += 32) {
        const double u = ej[m];
        el[m] = fma(-g, fma(-f1, u, ej1[m]), fma(-f, u, el[m]));
      }
    }
    jd = j + 1;
    fd = f1;
    pd = p1;
    __syncthreads();
  }
  if (jd >= 0 && x.warp == NW - 1) {
    double* el = X + jd * ld;
    const double* ej = X + (jd - 1) * ld;
    for (int m = x.lane; m < jd; m += 32) el[m] = fma(-fd, ej[m], el[m]);
    if (x.lane == 0) A[jd * ld + jd] = pd;
  }
  for (; j < k - 1; ++j) {  // a last single step (k - 1 odd)
    const double pj = A[j * ld + j];
    const double ip = rcp_nt64(pj > 1e-12 ? pj : 1e-12);
    for (int l = j + 1 + x.warp; l < k; l += NW) {
      const double f = A[j * ld + l] * ip;
      double* al = A + l * ld;
      const double* aj = A + j * ld;
      for (int m = l + x.lane; m < k; m += 32) al[m] = fma(-f, aj[m], al[m]);
      double* el = X + l * ld;
      const double* ej = X + j * ld;
      for (int m = x.lane; m <= j; m += 32) el[m] = fma(-f, ej[m], el[m]);
    }
  }
  __syncthreads();
  // X <- M = D E^T P^{-1/2}: M[m][i] = dsc[m] E[i][m] / sqrt(P_i) for m <= i (upper
  // triangular), built in A (only A's diagonal -- the pivots -- is still needed).
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
// Parallel cyclic Jacobi on H (k x k, smem, ld = kp + 1 with kp = k + (k & 1)),
// applied to the Rayleigh-Ritz basis directly: instead of accumulating V, each
// round's rotations are applied to the columns of nr row vectors QR (and SR),
// i.e. the CTA's own rows of Q (and S Q), staged in shared memory with stride
// ldr >= kp.  Round r of a sweep pairs (kp-1, r) and ((r+i) mod (kp-1),
// (r-i) mod (kp-1)), i = 1..kp/2-1 (circle method): kp/2 disjoint rotations.
// A round is two flat phases separated by barriers:
//   1. thread P < kp/2 computes the rotation of pair P (fp64);
//   2. H <- R H R^T by symmetric 2x2 blocks (pair P rows x pair P' columns,
//      P <= P', block and its mirror written), and the row vectors' columns
//      p, q rotated -- independent items over all threads.
// tau = (a_qq - a_pp) / (2 a_pq), t = sign(tau) / (|tau| + sqrt(1 + tau^2)),
// c = 1 / sqrt(1 + t^2), s = t c (Golub-Van Loan); c^2 + s^2 = 1 to rounding.
// On exit theta (smem) holds the eigenvalues in descending order and perm[c]
// the column of QR holding Ritz vector c.  Returns the sweeps used (-1:
// non-finite).  With nr = kp and QR = I the columns of QR are the eigenvectors.
__device__ int jacobi(const Ctx& x, double* H, int kin, int max_sweeps, double tol, double* theta,
                      int* perm, double* QR, double* SR, int nr, int ldr, long long* cyc = nullptr) {
  const int kp = kin + (kin & 1);
  const int ld = kp + 1;
  const int np = kp / 2;
  __shared__ double cs_c[kMaxBlock / 2 + 1], cs_s[kMaxBlock / 2 + 1];
  __shared__ int pp[kMaxBlock / 2 + 1], pq[kMaxBlock / 2 + 1];
  __shared__ int bad;
  __shared__ unsigned short tri[(kMaxBlock / 2 + 1) * (kMaxBlock / 2 + 2) / 2];
  long long c0 = 0, c1 = 0;
  const int ntri = np * (np + 1) / 2;
  for (int P = x.warp; P < np; P += NW)
    for (int P2 = P + x.lane; P2 < np; P2 += 32) {
      const int it = P * np - P * (P - 1) / 2 + (P2 - P);
      tri[it] = (unsigned short)((P << 8) | P2);
    }
  // dummy index for odd k: zero coupling, -inf diagonal (sorts last), zero column
  if (kin & 1) {
    for (int i = x.tid; i < kp; i += NT) {
      H[kin * ld + i] = (i == kin) ? -1e300 : 0.0;
      H[i * ld + kin] = (i == kin) ? -1e300 : 0.0;
    }
    for (int r = x.tid; r < nr; r += NT) {
      QR[r * ldr + kin] = 0.0;
      if (SR) SR[r * ldr + kin] = 0.0;
    }
  }
  __syncthreads();
  const double tol2 = tol * tol;
  const int nvi = np * nr;  // (pair, row) items of the row vectors
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    int any_sweep = 0;
    for (int round = 0; round < kp - 1; ++round) {
      if (cyc) c0 = clock64();
      int my_act = 0;
      if (x.tid < np) {
        const int P = x.tid;
        int p, q;
        if (P == 0) {
          p = kp - 1;
          q = round;
        } else {
          p = round + P;
          if (p >= kp - 1) p -= kp - 1;
          q = round - P;
          if (q < 0) q += kp - 1;
        }
        const double app = H[p * ld + p], aqq = H[q * ld + q], apq = H[p * ld + q];
        double c = 1.0, s = 0.0;
        if (apq != 0.0 && apq * apq > tol2 * fabs(app * aqq)) {
          // u = a_qq - a_pp, v = 2 a_pq, r = hypot(u, v), w = |u| / r = cos(2 theta):
          // c = sqrt((1 + w) / 2), s = sign(u) v / (2 r c)  (t = s / c is the smaller
          // root of t^2 + 2 tau t - 1 = 0, tau = u / v) -- two rsqrt, no division
          const double u = aqq - app, v = 2.0 * apq;
          const double ri = rsqrt_nt(fma(u, u, v * v));
          const double h = fma(0.5 * fabs(u), ri, 0.5);
          const double g = rsqrt_nt(h);  // 1 / c
          c = h * g;
          s = copysign(0.5, u) * v * ri * g;
          my_act = s != 0.0;
        }
        cs_c[P] = c;
        cs_s[P] = s;
        pp[P] = p;
        pq[P] = q;
      }
      const int any = __syncthreads_or(my_act);
      if (cyc) {
        c1 = clock64();
        cyc[0] += c1 - c0;
      }
      if (!any) continue;
      any_sweep = 1;
      // H blocks (P rows, P2 columns), P <= P2: B' = R_P B R_P2^T (flat triangle)
      for (int it = x.tid; it < ntri; it += NT) {
        const int P = tri[it] >> 8, P2 = tri[it] & 255;
        const double c = cs_c[P], s = cs_s[P];
        const double c2 = cs_c[P2], s2 = cs_s[P2];
        if (s == 0.0 && s2 == 0.0) continue;
        const int p = pp[P], q = pq[P], p2 = pp[P2], q2 = pq[P2];
        double* hp = H + p * ld;
        double* hq = H + q * ld;
        const double b00 = hp[p2], b01 = hp[q2], b10 = hq[p2], b11 = hq[q2];
        const double t00 = c * b00 - s * b10, t01 = c * b01 - s * b11;
        const double t10 = s * b00 + c * b10, t11 = s * b01 + c * b11;
        const double n00 = c2 * t00 - s2 * t01, n01 = s2 * t00 + c2 * t01;
        const double n10 = c2 * t10 - s2 * t11, n11 = s2 * t10 + c2 * t11;
        hp[p2] = n00;
        hp[q2] = n01;
        hq[p2] = n10;
        hq[q2] = n11;
        if (P2 != P) {
          H[p2 * ld + p] = n00;
          H[q2 * ld + p] = n01;
          H[p2 * ld + q] = n10;
          H[q2 * ld + q] = n11;
        }
      }
      // row vectors: columns p, q of every staged row <- (.) R_P^T
      for (int it = x.tid; it < nvi; it += NT) {
        const int P = it / nr, r = it - P * nr;
        const double s = cs_s[P];
        if (s == 0.0) continue;
        const double c = cs_c[P];
        double* qr = QR + r * ldr;
        const int p = pp[P], q = pq[P];
        const double a = qr[p], b = qr[q];
        qr[p] = c * a - s * b;
        qr[q] = s * a + c * b;
        if (SR) {
          double* sr = SR + r * ldr;
          const double u = sr[p], v = sr[q];
          sr[p] = c * u - s * v;
          sr[q] = s * u + c * v;
        }
      }
      __syncthreads();
      if (cyc) {
        c0 = clock64();
        cyc[1] += c0 - c1;
        cyc[5] += 1;
      }
    }
    if (!any_sweep) break;
  }
  // sort descending (stable by index)
  if (x.tid == 0) bad = 0;
  __syncthreads();
  if (x.tid < kin && !isfinite(H[x.tid * ld + x.tid])) bad = 1;
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

// Smallest eigenvalue of the m x m symmetric tridiagonal (alpha, beta[1..m-1]) by
// multisection: every thread evaluates the Sturm count at one point of the
// current bracket, the bracket shrinks to the first point with count >= 1 (3
// passes of NT points: (1/NT)^3 of the Gershgorin width).  All CTAs compute
// the same value.
__device__ double tridiag_min(const Ctx& x, const double* al, const double* be, int m) {
  __shared__ double lo, hi;
  __shared__ int first;
  if (x.tid == 0) {
    double l = 1e300, h = -1e300;
    for (int i = 0; i < m; ++i) {
      const double r = (i > 0 ? fabs(be[i]) : 0.0) + (i + 1 < m ? fabs(be[i + 1]) : 0.0);
      l = fmin(l, al[i] - r);
      h = fmax(h, al[i] + r);
    }
    lo = l;
    hi = h;
  }
  __syncthreads();
  for (int pass = 0; pass < 3; ++pass) {
    const double l = lo, h = hi;
    const double xv = l + (h - l) * (double)(x.tid + 1) / NT;
    int cnt = 0;
    double q = al[0] - xv;
    cnt += q < 0;
    for (int i = 1; i < m; ++i) {
      if (q == 0.0) q = 1e-300;
      q = al[i] - xv - be[i] * be[i] / q;
      cnt += q < 0;
    }
    if (x.tid == 0) first = NT;
    __syncthreads();
    if (cnt >= 1) atomicMin(&first, x.tid);
    __syncthreads();
    if (x.tid == 0) {
      const int f = first;
      hi = l + (h - l) * (double)(f + 1) / NT;
      lo = l + (h - l) * (double)f / NT;
    }
    __syncthreads();
  }
  const double r = 0.5 * (lo + hi);
  __syncthreads();
  return r;
}

// -------------------------------------------------------------- the solver --
__global__ void __launch_bounds__(NT, 1) k_eig_fused(FusedArgs P) {
  extern __shared__ __align__(128) double smem[];
  __shared__ double th[kMaxBlock + 2];    // Ritz values of the active block (indices nlock..)
  __shared__ double rs[kMaxBlock + 2];    // residuals
  __shared__ double thl[kMaxJ + 2];       // locked Ritz values
  __shared__ int perm[kMaxBlock + 2];
  __shared__ int src_of[kMaxBlock + 2];

  Ctx x;
  x.cta = blockIdx.x;
  x.G = gridDim.x;
  x.tid = threadIdx.x;
  x.warp = x.tid >> 5;
  x.lane = x.tid & 31;
  x.d = P.d;
  x.ls = P.ls;
  x.lb = P.lb;
  x.mv_m8 = P.mv_m8;
  x.mv_rb = P.mv_rb;
  x.mv_kb = P.mv_kb;
  x.mv_kc = P.mv_kc;
  const int d = P.d, J = P.J, k = P.k, LB = P.lb;
  const int R = (d + x.G - 1) / x.G;
  x.r0 = min(d, x.cta * R);
  x.r1 = min(d, x.r0 + R);
  const int kp = k + (k & 1);
  const int ld = kp + 1;
  x.r1s = smem;
  x.r2s = smem + region1_doubles(kp, R);
  x.sres = P.sres_off >= 0 ? smem + P.sres_off : nullptr;
  double* S = P.S;

  // buffer roles (indices into P.blk), swapped identically by every CTA
  int iQ = 0, iSQ = 1, iX = 2, iY = 3, iT = 4;
  auto B = [&](int i) { return P.blk[i]; };

  int nlock = 0, ka = k;
  int n_rr = 0, matvecs = 0, jsw = 0, breakdown = 0;
  double last_a = 0.0, last_b = 0.0;  // current damped interval (deflation shift = its centre)
  double a_lo = 0.0;                  // Lanczos estimate of lambda_min (0: none)
  double rprev = 1e-9;                // max relative residual after the last RR (Jacobi threshold)
  __shared__ long long pacc[8];
  long long pt = 0;
  if (x.tid < 8) pacc[x.tid] = 0;
  if (TK_EIG_PROFILE && x.tid == 0) pt = gtimer();
  // algorithmic fp64 flops of the solve (CTA 0 keeps the count; every CTA
  // executes the same control flow): products 2 d^2 n, Grams 2 d n_a n_b,
  // row-block applies 2 d m n, LDL^T CholQR (2/3) k^3, Jacobi rounds, deflation 4 d^2 n_l
  double flops = 0.0;
  long long mvt[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // CTA 0: product phase A, inner barrier, phase B,
                                                // leading barrier (ns); stage wait, compute, chunk loop (clk)
  auto tick = [&](int cat) {
    if (TK_EIG_PROFILE && x.cta == 0 && x.tid == 0) {
      const long long now = gtimer();
      pacc[cat] += now - pt;
      pt = now;
    }
  };

  zero_padding(x, S, P.rp, P.blk);
  gsync();
  load_sres(x, S);
  if (P.warm) copy_cols(x, P.basis, LB, B(iQ), LB, k);
  else fill_random(x, B(iQ), LB, k, P.seed);
  __syncthreads();

  auto mv = [&](const double* Y, double alpha, double* Out, double gamma, const double* Dm, double delta,
                const double* Em) {
    const bool prof = TK_EIG_PROFILE && x.cta == 0 && x.tid == 0;
    const long long tg0 = prof ? gtimer() : 0;
    gsync();  // Y, D, E (and S) complete
    if (prof) mvt[3] += gtimer() - tg0;
    matvec(x, P.mpart, S, Y, ka, alpha, Out, gamma, Dm, delta, Em,
           prof ? mvt : nullptr);  // own rows of Out on return
    ++matvecs;
    flops += 2.0 * d * d * ka;
    tick(PF_MV);
  };

  // ---- orthonormalise the active block against L and itself
  auto orth_active = [&](int passes, bool project) {
    if (nlock > 0 && project) {
      for (int pass = 0; pass < 2; ++pass) {
        gram_partial(x, P.L, J, nlock, B(iQ), LB, ka, P.part);
        reduce_bcast(x, P.part, nlock * ka, ka, P.red, x.r2s, ka);
        tick(PF_RED);
        flops += 4.0 * d * nlock * ka;
        // Q[own] -= L[own] Z  (Z = r2s, nlock x ka, ld ka)
        for (int r = x.r0 + x.warp; r < x.r1; r += NW)
          for (int c = x.lane; c < ka; c += 32) {
            double s = 0.0;
            for (int l = 0; l < nlock; ++l) s = fma(P.L[(int64_t)r * J + l], x.r2s[l * ka + c], s);
            B(iQ)[(int64_t)r * LB + c] -= s;
          }
        __syncthreads();
      }
    }
    const double shift = 11.0 * ((double)d * ka + (double)ka * (ka + 1)) * 1.1e-16 * ka;
    for (int pass = 0; pass < passes; ++pass) {
      gram_partial(x, B(iQ), LB, ka, B(iQ), LB, ka, P.part);
      reduce_bcast(x, P.part, ka * ka, ka, P.red, x.r1s, ld);
      tick(PF_RED);
      cholqr_factor(x, x.r1s, x.r2s, ka, ld, pass == 0 ? shift : 0.0);
      tick(PF_CHOL);
      flops += 2.0 * d * ka * ka + (2.0 / 3.0) * ka * ka * ka + 2.0 * d * ka * ka;
      apply_right(x, B(iQ), LB, ka, x.r2s, ld, 0, nullptr, B(iQ), LB, ka, x.r1s);
      tick(PF_APPLY);
    }
  };

  auto theta1 = [&]() {
    const double t = nlock > 0 ? thl[0] : th[0];
    return t > 0 ? t : 1.0;
  };

  // ---- Rayleigh-Ritz on the active block: Q <- Q V, SQ <- S Q V, th, rs
  auto rayleigh_ritz = [&]() {
    mv(B(iQ), 1.0, B(iSQ), 0.0, nullptr, 0.0, nullptr);
    gram_partial(x, B(iQ), LB, ka, B(iSQ), LB, ka, P.part);
    const int kk = ka + (ka & 1);
    reduce_bcast(x, P.part, ka * ka, ka, P.red, x.r1s, kk + 1);
    tick(PF_RED);
    for (int r = x.warp; r < ka; r += NW)
      for (int c = x.lane; c < ka; c += 32)
        if (r < c) {
          const double v = 0.5 * (x.r1s[r * (kk + 1) + c] + x.r1s[c * (kk + 1) + r]);
          x.r1s[r * (kk + 1) + c] = v;
          x.r1s[c * (kk + 1) + r] = v;
        }
    __syncthreads();
    // stage own rows of Q and SQ (region 2); the Jacobi rotations are applied to them
    const int nrr = x.r1 - x.r0;
    const int ldr = kk + 1;
    double* QR = x.r2s;
    double* SR = x.r2s + (size_t)nrr * ldr;
    for (int r = x.warp; r < nrr; r += NW)
      for (int c = x.lane; c < ka; c += 32) {
        QR[r * ldr + c] = B(iQ)[(int64_t)(x.r0 + r) * LB + c];
        SR[r * ldr + c] = B(iSQ)[(int64_t)(x.r0 + r) * LB + c];
      }
    __syncthreads();
    // rotation threshold: off-diagonals far below the current residual level
    // (rprev = max relative residual of the unconverged vectors after the last
    // RR) cannot matter yet; near convergence this is the strict 1e-13
    const double jtol = k == d ? 1e-15 : 1e-13;
    const int sw = jacobi(x, x.r1s, ka, k == d ? 60 : (n_rr == 0 ? P.jsweeps0 : P.jsweeps), jtol,
                          th + nlock, perm, QR, SR, nrr, ldr);
    tick(PF_JAC);
    if (sw < 0) breakdown = 1;
    else jsw += sw;
    {
      const double np2 = 0.5 * (ka + 1);
      flops += 2.0 * d * ka * ka  // H = Q^T S Q
               + (sw > 0 ? sw : 0) * (ka - 1) * (28.0 * np2 * (np2 + 1) / 2 + 12.0 * np2 * d);  // rotations
    }
    ++n_rr;
    // Q <- Q V, SQ <- SQ V: the rotated staged rows, columns in descending Ritz order
    for (int r = x.warp; r < nrr; r += NW)
      for (int c = x.lane; c < ka; c += 32) {
        B(iQ)[(int64_t)(x.r0 + r) * LB + c] = QR[r * ldr + perm[c]];
        B(iSQ)[(int64_t)(x.r0 + r) * LB + c] = SR[r * ldr + perm[c]];
      }
    __syncthreads();
    tick(PF_APPLY);
    // residual partials ||SQ_c - theta_c Q_c||^2 over own rows
    {
      const int nr = x.r1 - x.r0;
      for (int c = x.tid; c < ka; c += NT) {
        const double t = th[nlock + c];
        double s = 0.0;
        for (int r = 0; r < nr; ++r) {
          const int64_t o = (int64_t)(x.r0 + r) * LB + c;
          const double v = B(iSQ)[o] - t * B(iQ)[o];
          s = fma(v, v, s);
        }
        P.part[(size_t)c * x.G + x.cta] = s;  // entry-major
      }
    }
    reduce_bcast(x, P.part, ka, ka, P.red, rs + nlock, ka);
    tick(PF_RED);
    for (int c = x.tid; c < ka; c += NT) rs[nlock + c] = sqrt(rs[nlock + c]);
    __syncthreads();
    {
      const double t1 = theta1();
      double rm = 0.0;
      for (int i = nlock; i < J && i < nlock + ka; ++i) rm = fmax(rm, rs[i] / t1);
      rprev = rm;
    }
  };

  // deflate S by the locked columns [n0, n0 + nl) of L (LT holds S L), moving
  // them to eigenvalue sigma (the centre of the damped interval, so the filter
  // damps whatever components of them the active block regains):
  // S <- (I - Ln Ln^T) S (I - Ln Ln^T) + sigma Ln Ln^T = S - Ln W^T - W Ln^T,
  // W = P - Ln (Ln^T P) / 2 - sigma Ln / 2, P = S Ln
  auto deflate = [&](int n0, int nl) {
    const double sigma = last_b > 0 ? 0.5 * (last_a + last_b) : (a_lo > 0 ? a_lo : 0.0);
    // W and Ln stored transposed (nl x d; B(iX), B(iT) are scratch here: both
    // callers overwrite iT next), so the update's loads are coalesced over j
    double* WT = B(iX);
    double* LnT = B(iT);
    gram_partial(x, P.L + n0, J, nl, P.LT + n0, J, nl, P.part);
    reduce_bcast(x, P.part, nl * nl, nl, P.red, x.r2s, nl);
    tick(PF_RED);
    for (int r = x.r0 + x.warp; r < x.r1; r += NW)
      for (int c = x.lane; c < nl; c += 32) {
        double s = 0.0;
        for (int l = 0; l < nl; ++l) s = fma(P.L[(int64_t)r * J + n0 + l], x.r2s[l * nl + c], s);
        const double lv = P.L[(int64_t)r * J + n0 + c];
        WT[(int64_t)c * d + r] = P.LT[(int64_t)r * J + n0 + c] - 0.5 * s - 0.5 * sigma * lv;
        LnT[(int64_t)c * d + r] = lv;
      }
    gsync();  // W complete
    // S[own rows][j] -= sum_l Ln[r][l] W[j][l] + W[r][l] Ln[j][l], rows in chunks of 8
    double* lrs = x.r1s;           // [8][nl]
    double* wrs = x.r1s + 8 * nl;  // [8][nl]
    for (int rc = x.r0; rc < x.r1; rc += 8) {
      const int n8 = min(8, x.r1 - rc);
      for (int i = x.warp; i < 8; i += NW)
        for (int l = x.lane; l < nl; l += 32) {
          lrs[i * nl + l] = i < n8 ? P.L[(int64_t)(rc + i) * J + n0 + l] : 0.0;
          wrs[i * nl + l] = i < n8 ? __ldcg(WT + (int64_t)l * d + rc + i) : 0.0;
        }
      __syncthreads();
      for (int j = x.tid; j < d; j += NT) {
        double acc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.0;
        for (int l = 0; l < nl; ++l) {
          const double w = __ldcg(WT + (int64_t)l * d + j);
          const double lv = __ldcg(LnT + (int64_t)l * d + j);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = fma(lrs[i * nl + l], w, fma(wrs[i * nl + l], lv, acc[i]));
        }
        for (int i = 0; i < n8; ++i) S[(int64_t)(rc + i) * x.ls + j] -= acc[i];
      }
      __syncthreads();
    }
    gsync();
    load_sres(x, S);  // rows of other CTAs' tiles changed
    tick(PF_DEFL);
    flops += 4.0 * d * d * nl + 2.0 * d * nl * nl;
  };

  // move the converged leading active vectors into L (prefix, descending order)
  auto lock = [&]() {
    int nl = 0;
    const double th1 = theta1();
    while (nlock + nl < J && nl < ka && rs[nlock + nl] <= P.tol * th1) ++nl;
    if (nl == 0) return;
    copy_cols(x, B(iQ), LB, P.L + nlock, J, nl);
    copy_cols(x, B(iSQ), LB, P.LT + nlock, J, nl);
    for (int i = x.tid; i < nl; i += NT) thl[nlock + i] = th[nlock + i];
    __syncthreads();
    deflate(nlock, nl);
    const int kn = ka - nl;
    if (kn > 0) {  // compact the active block (row-local; same stride)
      copy_cols(x, B(iQ) + nl, LB, B(iT), LB, kn);
      copy_cols(x, B(iSQ) + nl, LB, B(iY), LB, kn);
      { int t = iQ; iQ = iT; iT = t; }
      { int t = iSQ; iSQ = iY; iY = t; }
    }
    __syncthreads();
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
    copy_cols(x, B(iQ), LB, pq_, 1, 1);
    gsync();
    for (int i = 0; i < npow; ++i) {
      matvec1(x, S, pq_, py_, P.part);
      ++matvecs;
      flops += 2.0 * d * d;
      gsync();
      const double nrm = allsum_scalar(x, P.part);
      const double inv = nrm > 0 ? rsqrt(nrm) : 0.0;
      for (int r = x.r0 + x.tid; r < x.r1; r += NT) pq_[r] = py_[r] * inv;
      gsync();
    }
    matvec1(x, S, pq_, py_, P.part);
    {
      double s = 0.0;
      for (int r = x.r0 + x.tid; r < x.r1; r += NT) s = fma(pq_[r], py_[r], s);
      block_partial(x, s, P.part + x.G);
    }
    gsync();
    const double th0 = allsum_scalar(x, P.part + x.G);
    {
      double s = 0.0;
      for (int r = x.r0 + x.tid; r < x.r1; r += NT) {
        const double v = py_[r] - th0 * pq_[r];
        s = fma(v, v, s);
      }
      block_partial(x, s, P.part + 2 * x.G);
    }
    gsync();
    const double r0v = sqrt(allsum_scalar(x, P.part + 2 * x.G));
    tick(PF_POW);
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
    const int kn = ka - 1;
    copy_cols(x, B(iQ) + 1, LB, B(iT), LB, kn);
    { int t = iQ; iQ = iT; iT = t; }
    __syncthreads();
    nlock = 1;
    ka = kn;
    orth_active(2, true);
    rayleigh_ritz();
    lock();
  };

  // lower end of the spectrum (Lanczos, 16 steps, no reorthogonalisation): the
  // Chebyshev filter then damps [lambda_min, theta_k] instead of [0, theta_k]
  if (!P.lanczos) a_lo = P.lmin_hint;
  if (P.lanczos) {
    constexpr int LZ = 16;
    __shared__ double lz_a[LZ], lz_b[LZ];
    double* v = P.pvec[0];
    double* vp = P.pvec[1];
    double* w = P.pvec[2];
    {
      double s0 = 0.0;
      for (int r = x.r0 + x.tid; r < x.r1; r += NT) {
        const uint64_t h = mix64(P.seed ^ 0x1a2c5ull ^ mix64((uint64_t)r * 2654435761ull));
        const double u = ((double)(h >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
        v[r] = u;
        vp[r] = 0.0;
        s0 = fma(u, u, s0);
      }
      block_partial(x, s0, P.part);
      gsync();
      const double inv = rsqrt(allsum_scalar(x, P.part));
      for (int r = x.r0 + x.tid; r < x.r1; r += NT) v[r] *= inv;
    }
    double beta = 0.0;
    for (int j = 0; j < LZ; ++j) {
      gsync();  // v complete
      // w = S v - beta vp (own rows); partials of v^T w and w^T w
      double pa = 0.0;
      for (int r = x.r0 + x.warp; r < x.r1; r += NW) {
        const double* srow = S + (int64_t)r * x.ls;
        double sacc = 0.0;
        for (int c = x.lane; c < d; c += 32) sacc = fma(__ldcg(srow + c), __ldcg(v + c), sacc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
        const double wr = sacc - beta * vp[r];
        if (x.lane == 0) {
          w[r] = wr;
          pa = fma(v[r], wr, pa);
        }
      }
      block_partial(x, pa, P.part);
      gsync();
      const double alpha = allsum_scalar(x, P.part);
      // w <- w - alpha v, beta_new = ||w|| (explicit: the shortcut ||w||^2 - alpha^2
      // cancels catastrophically next to an outlier eigenvalue)
      double pw = 0.0;
      for (int r = x.r0 + x.tid; r < x.r1; r += NT) {
        const double wr = w[r] - alpha * v[r];
        w[r] = wr;
        pw = fma(wr, wr, pw);
      }
      block_partial(x, pw, P.part + x.G);
      gsync();
      const double bnew = sqrt(allsum_scalar(x, P.part + x.G));
      if (x.tid == 0) {
        lz_a[j] = alpha;
        lz_b[j] = beta;  // beta_j couples j-1 and j
      }
      const double ib = bnew > 0 ? 1.0 / bnew : 0.0;
      for (int r = x.r0 + x.tid; r < x.r1; r += NT) {
        vp[r] = v[r];
        v[r] = w[r] * ib;
      }
      beta = bnew;
      ++matvecs;
      flops += 2.0 * d * d;
    }
    __syncthreads();
    a_lo = fmax(0.0, tridiag_min(x, lz_a, lz_b, LZ));
    tick(PF_POW);
    if (P.dbg && x.cta == 0 && x.tid == 0) printf("[eigf] lanczos lambda_min ~ %.6e\n", a_lo);
  }

  // an exact warm basis is the previous solve's orthonormal [L | Q]; a seeded
  // (fp32 hint + pseudo-random) or random block is orthonormalised first
  orth_active(P.warm_exact ? 0 : 2, true);
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
      // diagnostics: |L^T Q| and |SQ - S Q| (the state the filter starts from)
      gram_partial(x, P.L, J, nlock, B(iQ), LB, ka, P.part);
      reduce_bcast(x, P.part, nlock * ka, ka, P.red, x.r2s, ka);
      double m1 = 0.0;
      for (int e = x.tid; e < nlock * ka; e += NT) m1 = fmax(m1, fabs(x.r2s[e]));
      m1 = gmax(x, m1, P.part);
      mv(B(iQ), 1.0, B(iT), 0.0, nullptr, 0.0, nullptr);
      --matvecs;
      double m3 = 0.0;
      for (int r = x.r0; r < x.r1; ++r)
        for (int c = x.tid; c < ka; c += NT)
          m3 = fmax(m3, fabs(B(iT)[(int64_t)r * LB + c] - B(iSQ)[(int64_t)r * LB + c]));
      m3 = gmax(x, m3, P.part);
      if (x.cta == 0 && x.tid == 0)
        printf("[eigf-chk] outer=%d nlock=%d ka=%d |L^T Q|=%.3e |SQ - S Q|=%.3e\n", outer, nlock, ka, m1, m3);
    }
    const double th1 = theta1();
    const double thJ = th[J - 1];
    const double thtop = th[nlock];
    double b = th[k - 1];
    if (!(b > 0)) b = 1e-12 * th1;
    if (thJ <= b * (1 + 1e-12)) b = thJ * (1 - 1e-3);
    // damped interval [a, b]: a from Lanczos (minus 2 % of the width), else 0
    double a = a_lo > 0 ? a_lo - 0.02 * (b - a_lo) : 0.0;
    if (!(a > 0) || a > 0.9 * b) a = 0.0;
    last_b = b;
    last_a = a;
    const double e = (b - a) / 2, c = (b + a) / 2;
    const double xJ = fmax((thJ - c) / e, 1.0 + 1e-12);
    const double xt = fmax((thtop - c) / e, xJ);
    const double rJ = acosh(xJ), rt = acosh(xt);
    double rmax = 0;
    for (int i = nlock; i < J; ++i) rmax = fmax(rmax, rs[i] / th1);
    // total degree to reach tol (capped), in segments of <= m_amp degrees with an
    // orthonormalisation between them (T_m(x_top) <= 2e7 keeps CholQR in reach)
    int m_need = (int)ceil(log(fmax(rmax / P.tol, 4.0)) / fmax(rJ, 1e-6));
    const int m_amp = max(1, min(16, (int)floor(log(2e7) / fmax(rt, 1e-6))));
    m_need = max(1, min(min(m_need, 64), (m_amp < 6 ? 2 : 8) * m_amp));
    for (int done = 0; done < m_need;) {
      const int mseg = min(m_amp, m_need - done);
      // scaled Chebyshev recurrence (Zhou & Saad) damping [a, b], normalised at thtop
      double sigma = e / (thtop - c);
      const double tau = 2.0 / sigma;
      if (done > 0) mv(B(iQ), 1.0, B(iSQ), 0.0, nullptr, 0.0, nullptr);
      axpby(x, ka, LB, sigma / e, B(iSQ), -c * sigma / e, B(iQ), B(iY));
      int iXp = iQ, iYp = iY;
      int spare[2] = {iX, iT};
      int si = 0;
      for (int i = 2; i <= mseg; ++i) {
        const double sigma2 = 1.0 / (tau - sigma);
        const int iTp = spare[si];
        // T_i = 2 sigma2 / e (S T_{i-1} - c T_{i-1}) - sigma sigma2 T_{i-2}
        mv(B(iYp), 2 * sigma2 / e, B(iTp), -sigma * sigma2, B(iXp), -2 * sigma2 * c / e, B(iYp));
        spare[si] = iXp;
        si ^= 1;
        iXp = iYp;
        iYp = iTp;
        sigma = sigma2;
      }
      // the filtered block becomes Q (the five role indices stay a permutation)
      if (iYp != iQ) {
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
  for (int r = x.r0 + x.warp; r < x.r1; r += NW) {
    for (int j = x.lane; j < J; j += 32) {
      const int s = src_of[j];
      P.outV[(int64_t)r * J + j] = s < nlock ? P.L[(int64_t)r * J + s] : B(iQ)[(int64_t)r * LB + (s - nlock)];
    }
    // warm-start basis [L | A]
    for (int c = x.lane; c < k; c += 32)
      P.basis[(int64_t)r * LB + c] = c < nlock ? P.L[(int64_t)r * J + c] : B(iQ)[(int64_t)r * LB + (c - nlock)];
  }
  if (x.cta == 0) {
    for (int j = x.tid; j < J; j += NT) {
      const int s = src_of[j];
      P.theta_out[j] = s < nlock ? thl[s] : th[s];
    }
    if (x.tid < 8) P.prof[x.tid] += pacc[x.tid];
    if (x.tid == 0) {
      if (P.dbg) printf("[eigf-sync] grid barriers so far %llu, %.3f ms\n", g_gsync_stat[0], g_gsync_stat[1] * 1e-6);
      P.prof[8] += (long long)flops;
      for (int i = 0; i < 4; ++i) P.prof[9 + i] += mvt[i];
    }
    if (x.tid == 0) {
      P.dinfo[0] = P.lanczos ? a_lo : -1.0;  // -1: no new estimate
      P.dinfo[1] = last_b;
      P.info[0] = converged ? 1 : 0;
      P.info[1] = outer;
      P.info[2] = matvecs;
      P.info[3] = jsw;
      P.info[4] = breakdown;
    }
  }
}

// Unit-test kernel for the product on the padded layout (cooperative, all CTAs):
// Out = alpha S Y + gamma D, repeated `reps` times.
__global__ void __launch_bounds__(NT, 1) k_eigf_unit_mv(const double* S, const double* Y, int d, int n,
                                                       int ls, int lb, double alpha, double* Out,
                                                       double gamma, const double* D, double* mpart,
                                                       int reps, MvPlan pl) {
  extern __shared__ __align__(128) double smem[];
  Ctx x;
  x.cta = blockIdx.x;
  x.G = gridDim.x;
  x.tid = threadIdx.x;
  x.warp = x.tid >> 5;
  x.lane = x.tid & 31;
  x.d = d;
  const int R = (d + x.G - 1) / x.G;
  x.r0 = min(d, x.cta * R);
  x.r1 = min(d, x.r0 + R);
  x.ls = ls;
  x.lb = lb;
  x.mv_m8 = pl.m8;
  x.mv_rb = pl.RB;
  x.mv_kb = pl.KB;
  x.mv_kc = pl.kchunk;
  x.r1s = smem;
  x.r2s = smem;
  x.sres = nullptr;
  for (int i = 0; i < reps; ++i) {
    gsync();
    // reps == -2: two products into Out and Out + RP LB (determinism check)
    matvec(x, mpart, S, Y, n, alpha, Out, gamma, D, 0.0, nullptr);
  }
  if (reps == -2) {
    gsync();
    matvec(x, mpart, S, Y, n, alpha, Out, gamma, D, 0.0, nullptr);
    gsync();
    const int RP = (d + 63) / 64 * 64 + 64;
    matvec(x, mpart, S, Y, n, alpha, Out + (size_t)RP * lb, gamma, D, 0.0, nullptr);
  }
}

// Unit-test kernel for the k x k device routines (one CTA): mode 0 -> CholQR
// factor M of SPD `in` (out = M, k x k); mode 1 -> Jacobi (out = V with
// eigenvectors in columns, theta = eigenvalues descending, iout[0] = sweeps).
__global__ void __launch_bounds__(NT, 1) k_eigf_unit(int mode, const double* in, int k, double* out,
                                                    double* theta, int* iout, int sweeps, double shift) {
  extern __shared__ __align__(128) double smem[];
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
  x.ls = x.lb = 0;
  x.mv_m8 = x.mv_rb = x.mv_kb = x.mv_kc = 0;
  const int kp = k + (k & 1), ld = kp + 1;
  x.r1s = smem;
  x.r2s = smem + (size_t)kp * ld;
  x.sres = nullptr;
  for (int r = x.warp; r < k; r += NW)
    for (int c = x.lane; c < k; c += 32) x.r1s[r * ld + c] = in[r * k + c];
  __syncthreads();
  if (mode == 0) {
    cholqr_factor(x, x.r1s, x.r2s, k, ld, shift);
    for (int r = x.warp; r < k; r += NW)
      for (int c = x.lane; c < k; c += 32) out[r * k + c] = x.r2s[r * ld + c];
  } else {
    long long cyc[6] = {0, 0, 0, 0, 0, 0};
    double* QR = x.r2s;  // identity rows: the rotated rows are V
    for (int r = x.warp; r < kp; r += NW)
      for (int c = x.lane; c < kp; c += 32) QR[r * ld + c] = (r == c) ? 1.0 : 0.0;
    __syncthreads();
    const long long t0 = clock64();
    const int nrows = mode == 2 ? 8 : kp;  // mode 2: timing with a solver-like row count
    const int sw = jacobi(x, x.r1s, k, sweeps, 1e-13, th, perm, QR, mode == 2 ? QR + 8 * ld : nullptr, nrows, ld,
                          x.tid == 0 ? cyc : nullptr);
    const long long t1 = clock64();
    if (x.tid == 0) {
      for (int i = 0; i < 6; ++i) iout[1 + i] = (int)cyc[i];
      iout[7] = (int)(t1 - t0);
    }
    for (int r = x.warp; r < k; r += NW)
      for (int c = x.lane; c < k; c += 32) out[r * k + c] = QR[r * ld + perm[c]];
    for (int i = x.tid; i < k; i += NT) theta[i] = th[i];
    if (x.tid == 0) iout[0] = sw;
  }
}

// block size k = J + p: the oversampling p trades the k^3 Rayleigh-Ritz /
// CholQR work and the k-wide products against the convergence rate
// (theta_{k+1} / theta_J); measured on config 2, p ~ 10 minimises the solve time
int choose_block(int J, int64_t d, int oversample) {
  int k = J + (oversample > 0 ? oversample : std::max(8, std::min(J, 10)));
  if (k > kMaxBlock) k = kMaxBlock;
  if (k > d) k = (int)d;
  if (k & 1) k = (k + 1 <= kMaxBlock && k + 1 <= d) ? k + 1 : k - 1;
  if (k < J) k = J;
  return k;
}

int num_sms() {
  static int nsm = 0;
  if (nsm == 0) {
    int dev = 0;
    TK_CUDA(cudaGetDevice(&dev));
    TK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  }
  return nsm;
}

size_t product_smem(int d, int kmax, int G) {
  const MvPlan pl = mv_plan(d, G);
  return mv_smem_doubles(pl.m8, (kmax + 7) / 8) * sizeof(double);
}

size_t product_part_doubles(int d, int lb, int G) {
  const MvPlan pl = mv_plan(d, G);
  const int rpx = (d + 8 * pl.m8 - 1) / (8 * pl.m8) * (8 * pl.m8);
  return (size_t)pl.KB * rpx * lb;
}

void launch_unit_mv(const double* S, const double* Y, int d, int n, int ls, int lb, double alpha, double* O,
                    double gamma, const double* D, double* mpart, int reps, cudaStream_t st) {
  const int G = num_sms();
  const size_t smem = product_smem(d, n, G);
  smem_optin((const void*)k_eigf_unit_mv, smem);
  MvPlan pl = mv_plan(d, G);
  void* args[] = {&S, &Y, &d, &n, &ls, &lb, &alpha, &O, &gamma, &D, &mpart, &reps, &pl};
  TK_CUDA(cudaLaunchCooperativeKernel((const void*)k_eigf_unit_mv, dim3(G), dim3(NT), args, smem, st));
}

}  // namespace

void eig_layout(int64_t d, int64_t* ls, int64_t* rows) {
  const int64_t l = round_up(d, KCH);
  if (ls) *ls = l;
  if (rows) *rows = l + 64;
}

// working area (doubles) of the solver: max over its phases
size_t eig_work_doubles(int k, int d, int G) {
  const int kp = k + (k & 1);
  const int R = (d + G - 1) / G;
  const size_t r2 = std::max((size_t)kp * (kp + 1), (size_t)2 * R * (kp + 1));  // H, or staged Q/SQ rows
  const size_t jac = region1_doubles(kp, R) + r2;
  const size_t mv = product_smem(d, k, G) / sizeof(double);
  const size_t gp = (size_t)R * 2 * kp;
  return std::max(jac, std::max(mv, gp));
}
// resident S tile (doubles) of the product plan
size_t sres_doubles(int d, int G) {
  const MvPlan pl = mv_plan(d, G);
  return (size_t)16 * ((pl.m8 + 1) / 2) * (pl.kchunk + 4);
}
// dynamic smem budget: the device's per-block opt-in limit minus the solver's
// static shared memory (Jacobi tables, Ritz values: ~13.5 KB)
size_t smem_limit() {
  static size_t lim = 0;
  if (!lim) {
    int dev = 0, optin = 0;
    TK_CUDA(cudaGetDevice(&dev));
    TK_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa;
    TK_CUDA(cudaFuncGetAttributes(&fa, (const void*)k_eig_fused));
    lim = (size_t)optin - fa.sharedSizeBytes;
  }
  return lim;
}
#define SMEM_LIMIT smem_limit()

size_t eig_fused_smem(int k, int d, int G) {
  const size_t work = eig_work_doubles(k, d, G) * sizeof(double);
  const size_t sres = sres_doubles(d, G) * sizeof(double);
  return work + sres <= SMEM_LIMIT ? work + sres : work;
}

// Cold slot with a hint (the current factor, fp32 d x J row-major): the first J
// basis columns start from it, the k - J oversampling columns are a fixed
// pseudo-random fill (deterministic).
__global__ void k_seed_basis(double* __restrict__ basis, int64_t d, int LB, int k, const float* __restrict__ hint,
                             int J, uint64_t seed) {
  const int64_t n = d * LB;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / LB;
    const int c = (int)(e - r * LB);
    double v = 0.0;
    if (c < J) {
      v = (double)hint[r * J + c];
    } else if (c < k) {
      const uint64_t z = mix64(seed ^ ((uint64_t)r * 0x9E3779B97F4A7C15ull + (uint64_t)c));
      v = (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
    }
    basis[e] = v;
  }
}

bool eig_fused(double* S, int64_t d, int J, EigSlot& slot, EigWs& ws, const EigOpts& o, double* out_V,
               double* theta_dev, int* info_dev, cudaStream_t st, const float* hint) {
  const int k = choose_block(J, d, o.oversample);
  // one CTA per SM (cooperative: all co-resident); a small problem (d <= 256) runs on 32:
  // its products are latency-bound, and fewer CTAs make every grid barrier cheaper (measured
  // at config 4, d = 200: 63.6 ms of eigensolves per step on 148 CTAs, 56.7 ms on 32, 62.5 on 64)
  int grid = num_sms();
  if (d <= 256) grid = std::min(grid, 32);
  if (const char* e = std::getenv("TUCKER_EIG_GRID")) grid = std::max(1, std::min(num_sms(), std::atoi(e)));  // experiments
  const size_t smem = eig_fused_smem(k, (int)d, grid);
  if (smem > SMEM_LIMIT) fail(TUCKER_E_ARG, "eig_fused: block too large for shared memory");
  smem_optin((const void*)k_eig_fused, smem);
  {
    int per = 0;
    TK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_eig_fused, NT, smem));
    if (per < 1) fail(TUCKER_E_CUDA, "eig_fused: kernel cannot be resident");
  }
  int64_t LS = 0, RP = 0;
  eig_layout(d, &LS, &RP);
  const int LB = k + (k & 1);
  const size_t blk = (size_t)RP * LB + 64;
  ws.Q.ensure(blk);
  ws.SQ.ensure(blk);
  ws.X.ensure(blk);
  ws.Y.ensure(blk);
  ws.T.ensure(blk);
  ws.L.ensure((size_t)d * J);
  ws.LT.ensure((size_t)d * J);
  ws.fpart.ensure((size_t)grid * std::max<size_t>((size_t)k * k, 3));
  ws.fred.ensure((size_t)k * k);
  ws.pq.ensure((size_t)d);
  ws.py.ensure((size_t)d);
  ws.pz.ensure((size_t)d);
  ws.fprof.ensure(13);
  if (!ws.fprof_init) {
    TK_CUDA(cudaMemsetAsync(ws.fprof.p, 0, 13 * sizeof(long long), st));
    ws.fprof_init = true;
  }
  slot.basis.ensure((size_t)d * LB);
  ws.mpart.ensure(product_part_doubles((int)d, LB, grid));
  FusedArgs a;
  a.S = S;
  a.d = (int)d;
  a.J = J;
  a.k = k;
  a.ls = (int)LS;
  a.lb = LB;
  a.rp = (int)RP;
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
  a.pvec[2] = ws.pz.p;
  a.mpart = ws.mpart.p;
  {
    const MvPlan pl = mv_plan((int)d, grid);
    a.mv_m8 = pl.m8;
    a.mv_rb = pl.RB;
    a.mv_kb = pl.KB;
    a.mv_kc = pl.kchunk;
    const size_t work = eig_work_doubles(k, (int)d, grid);
    a.sres_off = (work + sres_doubles((int)d, grid)) * sizeof(double) <= SMEM_LIMIT ? (int)work : -1;
  }
  a.basis = slot.basis.p;
  a.warm = (slot.valid && slot.d == d && slot.k == k) ? 1 : 0;
  // an exact warm start reuses the last solve's orthonormal [L | Q] without the
  // initial CholQR; every 4th one re-orthonormalises so rounding drift cannot
  // accumulate over many sweeps
  a.warm_exact = a.warm && slot.exact_age < 4;
  slot.exact_age = a.warm_exact ? slot.exact_age + 1 : 0;
  if (!a.warm && hint) {  // cold slot: start from the caller's current factor
    TK_LAUNCH(k_seed_basis, 2 * grid, 256, 0, st, slot.basis.p, d, LB, k, hint, J,
              0x5eedb0000ull + (uint64_t)d * 131 + (uint64_t)J);
    a.warm = 1;
  }
  a.outV = out_V;
  a.theta_out = theta_dev;
  a.prof = ws.fprof.p;
  a.info = info_dev;
  a.dinfo = reinterpret_cast<double*>(info_dev + 8);
  // lambda_min only when it is worth it (first solve of the slot, or the last
  // estimate was a sizeable fraction of the filter bound), refreshed by Lanczos
  // every third solve; in between the last estimate minus 10 % of the interval
  // width (lambda_min drifts by a few % per sweep) is a safe lower bound
  const bool useful = !slot.valid || slot.lmin > 0.1 * slot.bval;
  a.lanczos = useful && (!slot.valid || slot.lz_age >= 2) ? 1 : 0;
  a.lmin_hint = (useful && !a.lanczos) ? slot.lmin - 0.1 * (slot.bval - slot.lmin) : 0.0;
  slot.lz_age = a.lanczos ? 0 : slot.lz_age + 1;
  a.tol = o.tol;
  if (const char* e = std::getenv("TUCKER_EIG_TOL")) a.tol = std::atof(e);  // experiments
  a.max_outer = o.max_outer;
  a.jsweeps = o.jacobi_sweeps;
  a.jsweeps0 = o.jacobi_sweeps_first;
  if (const char* e = std::getenv("TUCKER_EIG_JSW0")) a.jsweeps0 = std::atoi(e);  // experiments
  if (const char* e = std::getenv("TUCKER_EIG_JSW")) a.jsweeps = std::atoi(e);  // experiments
  a.seed = 0x5eed0000ull + (uint64_t)d * 131 + (uint64_t)J;
  static const bool dbg = std::getenv("TUCKER_EIG_DEBUG") != nullptr;
  a.dbg = dbg ? 1 : 0;
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
  // inputs are dense d x d / d x n device arrays; copy into the padded layout
  const int G = num_sms();
  int64_t LS = 0, RP = 0;
  eig_layout(d, &LS, &RP);
  const int LB = n + (n & 1);
  DBuf<double> dS((size_t)RP * LS), dY((size_t)RP * LB + 64), dD((size_t)RP * LB + 64),
      dO((size_t)RP * LB + 64), mp(product_part_doubles(d, LB, G));
  TK_CUDA(cudaMemsetAsync(dS.p, 0, dS.bytes(), st));
  TK_CUDA(cudaMemsetAsync(dY.p, 0, dY.bytes(), st));
  TK_CUDA(cudaMemsetAsync(dD.p, 0, dD.bytes(), st));
  TK_CUDA(cudaMemcpy2DAsync(dS.p, LS * 8, S, (size_t)d * 8, (size_t)d * 8, d, cudaMemcpyDeviceToDevice, st));
  TK_CUDA(cudaMemcpy2DAsync(dY.p, LB * 8, Y, (size_t)n * 8, (size_t)n * 8, d, cudaMemcpyDeviceToDevice, st));
  if (D)
    TK_CUDA(cudaMemcpy2DAsync(dD.p, LB * 8, D, (size_t)n * 8, (size_t)n * 8, d, cudaMemcpyDeviceToDevice, st));
  launch_unit_mv(dS.p, dY.p, d, n, (int)LS, LB, alpha, dO.p, D ? gamma : 0.0, dD.p, mp.p, 1, st);
  TK_CUDA(cudaMemcpy2DAsync(Out, (size_t)n * 8, dO.p, LB * 8, (size_t)n * 8, d, cudaMemcpyDeviceToDevice, st));
  TK_CUDA(cudaStreamSynchronize(st));
}

double eig_unit_mv_repeat(const double* S, const double* Y, int d, int n) {
  // two back-to-back products of the same (dense device) inputs: max |difference|
  const int G = num_sms();
  int64_t LS = 0, RP = 0;
  eig_layout(d, &LS, &RP);
  const int LB = n + (n & 1);
  DBuf<double> dS((size_t)RP * LS), dY((size_t)RP * LB + 64), dO(2 * (size_t)RP * LB + 64),
      mp(product_part_doubles(d, LB, G));
  TK_CUDA(cudaMemset(dS.p, 0, dS.bytes()));
  TK_CUDA(cudaMemset(dY.p, 0, dY.bytes()));
  TK_CUDA(cudaMemset(dO.p, 0, dO.bytes()));
  TK_CUDA(cudaMemcpy2D(dS.p, LS * 8, S, (size_t)d * 8, (size_t)d * 8, d, cudaMemcpyDeviceToDevice));
  TK_CUDA(cudaMemcpy2D(dY.p, LB * 8, Y, (size_t)n * 8, (size_t)n * 8, d, cudaMemcpyDeviceToDevice));
  launch_unit_mv(dS.p, dY.p, d, n, (int)LS, LB, 1.0, dO.p, 0.0, nullptr, mp.p, -2, 0);
  TK_CUDA(cudaDeviceSynchronize());
  std::vector<double> h(2 * (size_t)RP * LB);
  TK_CUDA(cudaMemcpy(h.data(), dO.p, h.size() * 8, cudaMemcpyDeviceToHost));
  double m = 0;
  for (int r = 0; r < d; ++r)
    for (int c = 0; c < n; ++c) m = std::max(m, std::fabs(h[(size_t)r * LB + c] - h[(size_t)RP * LB + (size_t)r * LB + c]));
  return m;
}

double eig_unit_mv_time(int d, int n, int reps) {
  const int G = num_sms();
  int64_t LS = 0, RP = 0;
  eig_layout(d, &LS, &RP);
  const int LB = n + (n & 1);
  DBuf<double> S((size_t)RP * LS), Y((size_t)RP * LB + 64), O((size_t)RP * LB + 64),
      mp(product_part_doubles(d, LB, G));
  TK_CUDA(cudaMemset(S.p, 0, S.bytes()));
  TK_CUDA(cudaMemset(Y.p, 0, Y.bytes()));
  cudaEvent_t a, b;
  TK_CUDA(cudaEventCreate(&a));
  TK_CUDA(cudaEventCreate(&b));
  // (T(1 + reps) - T(1)) / reps inside one cooperative launch (includes the two barriers)
  float ms1 = 0, ms2 = 0;
  TK_CUDA(cudaEventRecord(a, 0));
  launch_unit_mv(S.p, Y.p, d, n, (int)LS, LB, 1.0, O.p, 0.0, nullptr, mp.p, 1, 0);
  TK_CUDA(cudaEventRecord(b, 0));
  TK_CUDA(cudaEventSynchronize(b));
  TK_CUDA(cudaEventElapsedTime(&ms1, a, b));
  TK_CUDA(cudaEventRecord(a, 0));
  launch_unit_mv(S.p, Y.p, d, n, (int)LS, LB, 1.0, O.p, 0.0, nullptr, mp.p, 1 + reps, 0);
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
  smem_optin((const void*)k_eigf_unit, smem);
  TK_LAUNCH(k_eigf_unit, 1, NT, smem, st, mode, in, k, out, theta, iout, sweeps, shift);
}

}  // namespace tk
