// eig_small.cu -- all eigenvalues and the m leading eigenvectors of a small dense
// symmetric matrix (n <= 256), fp64: the Grams of BASELINE configs 1 and 4 (d = 100,
// 200) and config 3's Y^T Y route (d = 250), and the Rayleigh-Ritz problems of
// eig_large for blocks wider than the one-CTA Jacobi (k > 116).  Fig. 4 / Fig. 7
// "J leading eigenvectors" (MATLAB eigs P:1805).
//
// A direct method, so the cost does not depend on the eigengaps (MP's flat bulk cost
// the iterative solver ~175 products per solve at d = 200):
//   1. Householder tridiagonalisation Q^T S Q = T (k_tridiag): one thread-block cluster
//      of 4 CTAs, each holding a quarter of S's rows in shared memory; per column one
//      norm / vector exchange, one dot product and one vector exchange through
//      distributed shared memory (three cluster barriers), row-local rank-2 updates.
//   2. k_tri_eig (one CTA): the m largest eigenvalues of T by bisection on Sturm
//      counts (one thread per eigenvalue), their eigenvectors by inverse iteration with
//      a pivoted tridiagonal LU (one thread per vector, 3 iterations), modified
//      Gram-Schmidt among nearly equal eigenvalues (|l_i - l_j| <= 1e-9 ||T||: inverse
//      iterates of eigenvalues further apart are orthogonal to O(eps ||T|| / gap)), and the
//      back-transformation V = Q Y with the stored reflectors.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace tk {
namespace {

constexpr int kCl = 4;      // CTAs per cluster
constexpr int kNT = 512;    // threads per CTA
constexpr int kNMax = 256;  // largest n
constexpr int kRows = kNMax / kCl;

struct TriArgs {
  const double* S;  // n x n, row stride lds
  int64_t lds;
  int n;
  double* a;        // diagonal of T (n)
  double* e;        // off-diagonal of T (n - 1)
  double* H;        // Householder vectors: row k = u_k on entries k+1 .. n-1 (n x n)
  double* beta;     // H_k = I - beta_k u_k u_k^T (n)
};

__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kNT, 1) k_tridiag(TriArgs p) {
  extern __shared__ double Sr[];             // this CTA's rows of S (row stride kNMax), dynamic
  // exchange buffers, double buffered by step parity; every CTA pushes its part into all
  // CTAs' copies (remote shared-memory stores) before the cluster barrier, so after it
  // every read is local
  __shared__ double ub[2][kNMax], qb[2][kNMax];
  __shared__ double nrm[2][kCl], kpart[2][kCl];
  __shared__ double wred[kNT / 32];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int n = p.n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (n + kCl - 1) / kCl;
  const int r0 = rank * per, r1 = min(n, r0 + per);
  const int nr = max(0, r1 - r0);
  for (int r = warp; r < nr; r += kNT / 32)
    for (int c = lane; c < n; c += 32) Sr[r * kNMax + c] = p.S[(int64_t)(r0 + r) * p.lds + c];
  double* ubr[kCl];
  double* qbr[kCl];
  double* nrr[kCl];
  double* kpr[kCl];
  for (int c = 0; c < kCl; ++c) {
    ubr[c] = cl.map_shared_rank(&ub[0][0], c);
    qbr[c] = cl.map_shared_rank(&qb[0][0], c);
    nrr[c] = cl.map_shared_rank(&nrm[0][0], c);
    kpr[c] = cl.map_shared_rank(&kpart[0][0], c);
  }
  __syncthreads();
  // CTA-wide sum of one value per thread (warp shuffles + one shared-memory pass)
  auto csum = [&](double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) wred[warp] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kNT / 32; ++w) s += wred[w];
    return s;  // the caller's next barrier orders wred's reuse
  };
  for (int k = 0; k < n - 2; ++k) {
    const int b = k & 1;
    // 1. own part of x = S[k+1.., k] and its partial ||x||^2, pushed to every CTA
    double ss = 0.0;
    for (int r = tid; r < nr; r += kNT) {
      const int i = r0 + r;
      const double x = i > k ? Sr[r * kNMax + k] : 0.0;
      ss += x * x;
#pragma unroll
      for (int c = 0; c < kCl; ++c) ubr[c][b * kNMax + i] = x;
    }
    ss = csum(ss);
    if (tid < kCl) nrr[tid][b * kCl + rank] = ss;
    cl.sync();
    double nx2 = 0.0;
#pragma unroll
    for (int c = 0; c < kCl; ++c) nx2 += nrm[b][c];
    const double* u = ub[b];
    const double x0 = u[k + 1];
    const double nx = sqrt(nx2);
    const double alpha = x0 >= 0 ? -nx : nx;
    const double uu = 2.0 * (nx2 - alpha * x0);  // u^T u with u = x - alpha e_{k+1}
    const double beta = uu > 0 ? 2.0 / uu : 0.0;
    const double u1 = x0 - alpha;                  // u[k + 1] (u[] itself keeps x0)
    // 2. p = beta S_sub u (own rows; warp per row), partial K = (beta / 2) u^T p
    double kp = 0.0;
    for (int r = warp; r < nr; r += kNT / 32) {
      const int i = r0 + r;
      double s = 0.0;
      if (i > k) {
        for (int j = k + 1 + lane; j < n; j += 32) s = fma(Sr[r * kNMax + j], j == k + 1 ? u1 : u[j], s);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
          const double ui = i == k + 1 ? u1 : u[i];
          qb[b][i] = beta * s;  // p_i, own rows
          kp += beta * s * ui;
        }
      }
    }
    kp = csum(kp);
    if (tid < kCl) kpr[tid][b * kCl + rank] = kp;
    cl.sync();
    double K = 0.0;
#pragma unroll
    for (int c = 0; c < kCl; ++c) K += kpart[b][c];
    K *= 0.5 * beta;
    // 3. q = p - K u (own rows), pushed to every CTA
    for (int r = tid; r < nr; r += kNT) {
      const int i = r0 + r;
      if (i > k) {
        const double qi = qb[b][i] - K * (i == k + 1 ? u1 : u[i]);
#pragma unroll
        for (int c = 0; c < kCl; ++c) qbr[c][b * kNMax + i] = qi;
      }
    }
    // bookkeeping while the exchange completes
    if (rank == 0) {
      for (int j = tid; j < n; j += kNT) p.H[(int64_t)k * n + j] = j > k ? (j == k + 1 ? u1 : u[j]) : 0.0;
      if (tid == 0) {
        p.beta[k] = beta;
        p.e[k] = alpha;
      }
    }
    if (k >= r0 && k < r1 && tid == 0) p.a[k] = Sr[(k - r0) * kNMax + k];
    cl.sync();
    // 4. S_sub -= u q^T + q u^T on own rows (warp per row, lanes over columns)
    const double* q = qb[b];
    for (int r = warp; r < nr; r += kNT / 32) {
      const int i = r0 + r;
      if (i <= k) continue;
      const double ui = i == k + 1 ? u1 : u[i], qi = q[i];
      for (int j = k + 1 + lane; j < n; j += 32)
        Sr[r * kNMax + j] -= ui * q[j] + qi * (j == k + 1 ? u1 : u[j]);
    }
    __syncthreads();
  }
  // the trailing 2 x 2 (or 1 x 1) block
  for (int i = max(0, n - 2); i < n; ++i)
    if (i >= r0 && i < r1 && tid == 0) {
      p.a[i] = Sr[(i - r0) * kNMax + i];
      if (i == n - 2) p.e[i] = Sr[(i - r0) * kNMax + i + 1];
    }
  if (rank == 0)
    for (int k = max(0, n - 2); k < n; ++k) {
      for (int j = tid; j < n; j += kNT) p.H[(int64_t)k * n + j] = 0.0;
      if (tid == 0) p.beta[k] = 0.0;
    }
  cl.sync();  // no CTA leaves while others may still write into its shared memory
}

// number of eigenvalues of T (diag a, off-diagonal e) below x (Sturm sequence)
__device__ int sturm_count(const double* a, const double* e, int n, double x, double tiny) {
  int cnt = 0;
  double qv = a[0] - x;
  if (fabs(qv) < tiny) qv = -tiny;
  if (qv < 0) ++cnt;
  for (int i = 1; i < n; ++i) {
    qv = (a[i] - x) - e[i - 1] * e[i - 1] / qv;
    if (fabs(qv) < tiny) qv = -tiny;
    if (qv < 0) ++cnt;
  }
  return cnt;
}

// one CTA: m leading eigenpairs of T, back-transformed with the reflectors
__global__ void __launch_bounds__(256) k_tri_eig(const double* __restrict__ a, const double* __restrict__ e, int n,
                                                 const double* __restrict__ H, const double* __restrict__ beta, int m,
                                                 double* __restrict__ Y /* m x n scratch */,
                                                 double* __restrict__ F /* m x 5 n scratch */,
                                                 double* __restrict__ V /* n x m, ld m */, double* __restrict__ theta,
                                                 int* __restrict__ info) {
  __shared__ double lam[kNMax];
  __shared__ double red[8];
  __shared__ double sa[kNMax], se[kNMax];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < n; i += blockDim.x) {
    sa[i] = a[i];
    se[i] = i < n - 1 ? e[i] : 0.0;
  }
  __syncthreads();
  // Gershgorin interval and scale
  double lo = sa[0], hi = sa[0], tn = 0.0;
  for (int i = 0; i < n; ++i) {
    const double r = (i > 0 ? fabs(se[i - 1]) : 0.0) + (i < n - 1 ? fabs(se[i]) : 0.0);
    lo = fmin(lo, sa[i] - r);
    hi = fmax(hi, sa[i] + r);
    tn = fmax(tn, fabs(sa[i]) + r);
  }
  const double tiny = 1e-300 + 1e-30 * tn;
  // multisection: a warp per eigenvalue j (descending = the (n - 1 - j)-th smallest); each
  // round its 32 lanes evaluate Sturm counts at 31 interior points of [l, h] (5 bits per round)
  for (int j = warp; j < m; j += (int)(blockDim.x >> 5)) {
    const int kth = n - 1 - j;
    double l = lo - 1e-12 * tn - tiny, h = hi + 1e-12 * tn + tiny;
    for (int it = 0; it < 16 && h - l > 2.2e-16 * fmax(fabs(l), fabs(h)) + tiny; ++it) {
      const double x = l + (h - l) * (double)(lane + 1) / 32.0;
      const bool below = lane < 31 && sturm_count(sa, se, n, x, tiny) <= kth;  // x still left of the target
      const unsigned bal = __ballot_sync(0xffffffffu, below);
      const int nb = __popc(bal);  // points 1..nb are <= the target: new interval [x_nb, x_{nb+1}]
      const double nl = nb > 0 ? l + (h - l) * (double)nb / 32.0 : l;
      const double nh = l + (h - l) * (double)(nb + 1) / 32.0;
      l = nl;
      h = nh;
    }
    if (lane == 0) lam[j] = 0.5 * (l + h);
  }
  __syncthreads();
  // inverse iteration, one thread per eigenvector (pivoted tridiagonal LU of T - lambda I)
  const double eps = 2.2e-16;
  for (int j = tid; j < m; j += blockDim.x) {
    double* y = Y + (size_t)j * n;
    double* dl = F + (size_t)j * 5 * n;
    double* dd = dl + n;
    double* du = dd + n;
    double* du2 = du + n;
    double* pv = du2 + n;  // 1.0 = rows i, i+1 swapped
    // a tiny shift separates equal eigenvalues; starting vector: fixed pseudo-random
    const double shift = lam[j] + eps * tn * (1.0 + 0.25 * (j & 7));
    for (int i = 0; i < n; ++i) {
      dd[i] = sa[i] - shift;
      du[i] = se[i];
      dl[i] = se[i];
      du2[i] = 0.0;
      pv[i] = 0.0;
      uint64_t z = (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull ^ (uint64_t)(j + 7) * 0xBF58476D1CE4E5B9ull;
      z ^= z >> 31;
      y[i] = 0.5 + (double)(z >> 11) * (1.0 / 9007199254740992.0);
    }
    for (int i = 0; i < n - 1; ++i) {
      if (fabs(dd[i]) >= fabs(dl[i])) {
        if (dd[i] == 0.0) dd[i] = eps * tn + tiny;
        const double f = dl[i] / dd[i];
        dl[i] = f;
        dd[i + 1] -= f * du[i];
      } else {
        const double f = dd[i] / dl[i];
        dd[i] = dl[i];
        dl[i] = f;
        const double t = du[i];
        du[i] = dd[i + 1];
        dd[i + 1] = t - f * dd[i + 1];
        if (i < n - 2) {
          du2[i] = du[i + 1];
          du[i + 1] = -f * du[i + 1];
        }
        pv[i] = 1.0;
      }
    }
    if (dd[n - 1] == 0.0) dd[n - 1] = eps * tn + tiny;
    for (int it = 0; it < 3; ++it) {
      for (int i = 0; i < n - 1; ++i) {  // L
        if (pv[i] == 0.0) {
          y[i + 1] -= dl[i] * y[i];
        } else {
          const double t = y[i];
          y[i] = y[i + 1];
          y[i + 1] = t - dl[i] * y[i + 1];
        }
      }
      y[n - 1] /= dd[n - 1];  // U
      if (n > 1) y[n - 2] = (y[n - 2] - du[n - 2] * y[n - 1]) / dd[n - 2];
      for (int i = n - 3; i >= 0; --i) y[i] = (y[i] - du[i] * y[i + 1] - du2[i] * y[i + 2]) / dd[i];
      double s = 0.0;
      for (int i = 0; i < n; ++i) s = fma(y[i], y[i], s);
      s = 1.0 / sqrt(s);
      for (int i = 0; i < n; ++i) y[i] *= s;
    }
  }
  __syncthreads();
  // modified Gram-Schmidt among close eigenvalues (twice), the whole CTA per dot product
  auto csum = [&](double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    __syncthreads();
    return s;
  };
  for (int j = 1; j < m; ++j) {
    int i0 = j;
    while (i0 > 0 && lam[i0 - 1] - lam[i0] <= 1e-9 * tn) --i0;
    if (i0 == j) continue;
    double* yj = Y + (size_t)j * n;
    for (int pass = 0; pass < 2; ++pass) {
      for (int i = i0; i < j; ++i) {
        const double* yi = Y + (size_t)i * n;
        double s = 0.0;
        for (int r = tid; r < n; r += blockDim.x) s = fma(yi[r], yj[r], s);
        s = csum(s);
        for (int r = tid; r < n; r += blockDim.x) yj[r] -= s * yi[r];
        __syncthreads();
      }
      double s = 0.0;
      for (int r = tid; r < n; r += blockDim.x) s = fma(yj[r], yj[r], s);
      s = 1.0 / sqrt(csum(s));
      for (int r = tid; r < n; r += blockDim.x) yj[r] *= s;
      __syncthreads();
    }
  }
  // back-transformation: x = H_0 H_1 .. H_{n-3} y (reflectors applied last to first)
  for (int k = n - 3; k >= 0; --k) {
    const double* uk = H + (size_t)k * n;
    const double bk = beta[k];
    if (bk == 0.0) continue;
    // warp w handles the vectors j = w, w + 8, ...: dot product, then the update
    for (int j = warp; j < m; j += (int)(blockDim.x >> 5)) {
      double* yj = Y + (size_t)j * n;
      double s = 0.0;
      for (int r = k + 1 + lane; r < n; r += 32) s = fma(uk[r], yj[r], s);
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      s *= bk;
      for (int r = k + 1 + lane; r < n; r += 32) yj[r] -= s * uk[r];
    }
    __syncwarp();
  }
  __syncthreads();
  for (int e2 = tid; e2 < n * m; e2 += blockDim.x) {
    const int r = e2 / m, j = e2 - r * m;
    V[(size_t)r * m + j] = Y[(size_t)j * n + r];
  }
  for (int j = tid; j < m; j += blockDim.x) theta[j] = lam[j];
  if (tid < 8) info[tid] = tid == 0 || tid == 1 ? 1 : 0;  // converged (direct method), 1 "iteration"
  if (tid == 0) {
    double* dv = reinterpret_cast<double*>(info + 8);
    dv[0] = -1.0;  // no Lanczos / filter-bound estimates (eig_check keeps the slot's)
    dv[1] = -1.0;
  }
}


// ---------------------------------------------------------------------------
// k_eig_direct: the whole direct solve in ONE CTA of 1024 threads for n small
// enough that the packed lower triangle of S (n (n + 1) / 2 doubles; n = 200:
// 161 KB) fits in shared memory -- no cluster barriers, no DSMEM, no global
// round trips inside the sequential parts (the 4-CTA path above measured ~4 ms
// at n = 200, dominated by those).  Phases:
//   1. Householder tridiagonalisation Q^T S Q = T on the packed triangle: per
//      column k two block barriers; lane l owns the indices j = l + 32 m (its u_j
//      and q_j live in registers), warp w the rows i = k + 1 + w + 32 r; the
//      symmetric product p = beta S u reads the row part (j <= i) and the column
//      part (j > i) of the packed storage, the rank-2 update S -= u q^T + q u^T
//      rewrites the row part; the lane that owns j = k + 1 also emits the next
//      column (and its norm) so it is ready after the barrier.  The reflectors
//      go to global memory (rows of H) for phase 4.
//   2. Eigenvalues m largest of T (scaled by its Gershgorin bound) by
//      multisection: a warp per eigenvalue, 32 points per round (11 rounds:
//      33^-11 ~ 2e-17 of the interval), Sturm counts by the division-free
//      three-term recurrence of the leading principal minors (sign changes;
//      rescaled when they leave [1e-150, 1e150]).
//   3. Eigenvectors by inverse iteration (one thread per vector, pivoted LU of
//      T - lambda I in shared memory, 3 iterations; a tiny shift per vector and
//      a fixed pseudo-random start separate equal eigenvalues), modified
//      Gram-Schmidt (twice) among eigenvalues closer than 1e-9 ||T||.
//   4. Back-transformation V = H_0 .. H_{n-3} Y, a warp per vector.
// ---------------------------------------------------------------------------
constexpr int kDT = 1024;
constexpr int kDW = kDT / 32;
constexpr int kDJ = 7;  // indices per lane: n <= 224

struct DirArgs {
  const double* S;
  int64_t lds;
  int n, m;
  int ws;       // doubles of dynamic shared memory
  double* H;    // n x n: row k = reflector u_k (entries k + 1 .. n - 1)
  double* V;    // n x m, ld m
  double* theta;
  int* info;
  unsigned long long* prof;  // nullable: per-phase globaltimer stamps (TUCKER_EIG_PROF, tools)
  int dbg;                   // TUCKER_EIG_DBG (timing experiments; wrong results): 1 skip phase 2, 2 skip phase 1
};

__device__ __forceinline__ void stamp(unsigned long long* prof, int slot) {
  if (prof != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    prof[slot] = t;
  }
}

__device__ __forceinline__ int pidx(int i, int j) { return (i * (i + 1)) / 2 + j; }
__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// phases 2-4 of the direct solve: T = (sa, se) (overwritten: scaled), reflectors in rows of H
// (u_k on entries k + 1 .. n - 1; beta_k in H[k][k], or beta[k] when beta != nullptr), a
// shared-memory workspace L of wsz doubles; V (n x m, ld m), theta (m), info record
__device__ void eig_tail(int n, int m, double* sa, double* se, double* te2, double* L, int wsz, double* lam,
                         double* red, const double* Hg, const double* betag, double* Vout, double* theta_out,
                         int* info_out, unsigned long long* prof = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- 2. eigenvalues: scale T by its Gershgorin bound tn
  double tn = 0.0;  // max_i |a_i| + |e_i-1| + |e_i|: per-thread maxima, warp max, then the 32 warp maxima
  for (int i = tid; i < n; i += kDT) tn = fmax(tn, fabs(sa[i]) + (i > 0 ? fabs(se[i - 1]) : 0.0) + (i < n - 1 ? fabs(se[i]) : 0.0));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tn = fmax(tn, __shfl_xor_sync(0xffffffffu, tn, o));
  if (lane == 0) red[warp] = tn;
  __syncthreads();
  tn = red[lane];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tn = fmax(tn, __shfl_xor_sync(0xffffffffu, tn, o));
  const double sc = tn > 0 ? 1.0 / tn : 1.0;
  __syncthreads();
  for (int i = tid; i < n; i += kDT) {
    sa[i] *= sc;
    se[i] *= sc;
    te2[i] = se[i] * se[i];
  }
  __syncthreads();
  for (int j = warp; j < m; j += kDW) {
    const int kth = n - 1 - j;  // the (n - 1 - j)-th smallest
    double l = -1.0 - 1e-12, h = 1.0 + 1e-12;
    for (int it = 0; it < 7; ++it) {  // 33^-7 ~ 2e-11 of the interval: the shift of inverse iteration
      const double x = l + (h - l) * (double)(lane + 1) / 33.0;
      // sign changes of the leading minors p_0 = 1, p_1 = a_0 - x, p_i = (a_{i-1} - x) p_{i-1} - e_{i-2}^2 p_{i-2}
      // (T is scaled to ||T|| <= 1, so |p| grows by <= 3 per step: rescaled every 8 steps when it
      // leaves [1e-100, 1e100]; an exact zero minor counts as a sign change, like a -0 pivot)
      int cnt = 0;
      double pm = 1.0, pc = sa[0] - x;
      bool neg = pc <= 0.0;  // p_0 = 1 > 0; a zero p_1 counts as negative
      cnt += neg;
      int i = 1;
      for (; i + 8 <= n; i += 8) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const double pn = fma(sa[i + r] - x, pc, -te2[i + r - 1] * pm);
          // sign of a zero minor: opposite to its predecessor's (a -0 pivot); kept off the chain
          const bool ng = pn == 0.0 ? !neg : pn < 0.0;
          cnt += ng != neg;
          neg = ng;
          pm = pc;
          pc = pn;
        }
        const double an = fabs(pc);
        if (an > 1e100 || an < 1e-100) {
          const double f = an > 1e100 ? 1e-100 : 1e100;
          pc *= f;
          pm *= f;
        }
      }
      for (; i < n; ++i) {
        const double pn = fma(sa[i] - x, pc, -te2[i - 1] * pm);
        const bool ng = pn == 0.0 ? !neg : pn < 0.0;
        cnt += ng != neg;
        neg = ng;
        pm = pc;
        pc = pn;
      }
      const unsigned below = __ballot_sync(0xffffffffu, cnt <= kth);
      const int nb = __popc(below);  // points 0 .. nb - 1 lie at or left of the target
      const double nl = nb > 0 ? l + (h - l) * (double)nb / 33.0 : l;
      const double nh = l + (h - l) * (double)(nb + 1) / 33.0;
      l = nl;
      h = nh;
    }
    if (lane == 0) lam[j] = 0.5 * (l + h);
  }
  __syncthreads();
  stamp(prof, 3);
  // ---- 3. inverse iteration; workspace: Y [n][m] | per round R vectors x (dl, dd, du, du2) [n][R] | pv bytes [n][R]
  double* Y = L;
  const int R = max(1, min(m, (int)((wsz - n * m) / (4 * n + (n + 7) / 8 + 1))));
  double* dl = Y + n * m;
  double* dd = dl + n * R;
  double* du = dd + n * R;
  double* du2 = du + n * R;
  unsigned char* pv = reinterpret_cast<unsigned char*>(du2 + n * R);
  const double eps = 2.2e-16;
  for (int j0 = 0; j0 < m; j0 += R) {
    const int t = tid;
    const int j = j0 + t;
    if (t < R && j < m) {
      const double shift = lam[j] + eps * (1.0 + 0.25 * (j & 7));
#define AT(a, i) a[(i) * R + t]
      // pivoted LU of T - shift I (LAPACK dgttrf's elimination), the current row carried in registers
      double cd = sa[0] - shift, cu = n > 1 ? se[0] : 0.0;
      for (int i = 0; i < n - 1; ++i) {
        const double li = se[i], nd = sa[i + 1] - shift, nu = i + 1 < n - 1 ? se[i + 1] : 0.0;
        if (fabs(cd) >= fabs(li)) {
          const double dv = cd == 0.0 ? eps : cd;
          const double rv = 1.0 / dv;
          const double f = li * rv;
          AT(dl, i) = f;
          AT(dd, i) = rv;
          AT(du, i) = cu;
          AT(du2, i) = 0.0;
          pv[i * R + t] = 0;
          cd = fma(-f, cu, nd);
          cu = nu;
        } else {
          const double rl = 1.0 / li;
          const double f = cd * rl;
          AT(dl, i) = f;
          AT(dd, i) = rl;
          AT(du, i) = nd;
          AT(du2, i) = nu;
          pv[i * R + t] = 1;
          cd = fma(-f, nd, cu);
          cu = -f * nu;
        }
      }
      AT(dd, n - 1) = 1.0 / (cd == 0.0 ? eps : cd);
      // start vector: fixed pseudo-random, in [0.5, 1)
      for (int i = 0; i < n; ++i) {
        uint64_t z = (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull ^ (uint64_t)(j + 7) * 0xBF58476D1CE4E5B9ull;
        z ^= z >> 31;
        Y[i * m + j] = 0.5 + (double)(z >> 11) * (1.0 / 9007199254740992.0);
      }
      // the solves read 8 steps' operands into registers before computing them (no load waits
      // behind the previous step's store: the chain is the register recurrence only)
      for (int it = 0; it < 2; ++it) {
        double cy = Y[j];  // forward: L (row swaps as recorded)
        int i = 0;
        for (; i + 8 <= n - 1; i += 8) {
          double ny[8], fv[8];
          bool sw[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            ny[u] = Y[(i + u + 1) * m + j];
            fv[u] = AT(dl, i + u);
            sw[u] = pv[(i + u) * R + t] != 0;
          }
          double out[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            out[u] = sw[u] ? ny[u] : cy;
            cy = sw[u] ? fma(-fv[u], ny[u], cy) : fma(-fv[u], cy, ny[u]);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) Y[(i + u) * m + j] = out[u];
        }
        for (; i < n - 1; ++i) {
          const double ny = Y[(i + 1) * m + j], f = AT(dl, i);
          if (!pv[i * R + t]) {
            Y[i * m + j] = cy;
            cy = fma(-f, cy, ny);
          } else {
            Y[i * m + j] = ny;
            cy = fma(-f, ny, cy);
          }
        }
        // backward: U (reciprocal pivots), y_{i+1}, y_{i+2} carried
        double y1 = cy * AT(dd, n - 1), y2 = 0.0;
        Y[(n - 1) * m + j] = y1;
        double ssq = y1 * y1;
        i = n - 2;
        for (; i >= 7; i -= 8) {
          double yv[8], uv1[8], uv2[8], rv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            yv[u] = Y[(i - u) * m + j];
            uv1[u] = AT(du, i - u);
            uv2[u] = AT(du2, i - u);
            rv[u] = AT(dd, i - u);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const double yi = (yv[u] - uv1[u] * y1 - uv2[u] * y2) * rv[u];
            yv[u] = yi;
            ssq = fma(yi, yi, ssq);
            y2 = y1;
            y1 = yi;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) Y[(i - u) * m + j] = yv[u];
        }
        for (; i >= 0; --i) {
          const double yi = (Y[i * m + j] - AT(du, i) * y1 - AT(du2, i) * y2) * AT(dd, i);
          Y[i * m + j] = yi;
          ssq = fma(yi, yi, ssq);
          y2 = y1;
          y1 = yi;
        }
        const double sN = 1.0 / sqrt(ssq);
        for (int i2 = 0; i2 < n; ++i2) Y[i2 * m + j] *= sN;
      }
      // the eigenvalue as the Rayleigh quotient y^T T y of the converged vector (the bisection
      // bracket is only ~2e-11 ||T|| narrow; the quotient's error is O(residual^2))
      {
        double rq = 0.0, yp = Y[j];
        for (int i2 = 0; i2 < n; ++i2) {
          const double yn = i2 + 1 < n ? Y[(i2 + 1) * m + j] : 0.0;
          rq = fma(yp, fma(sa[i2], yp, 2.0 * se[i2] * yn), rq);
          yp = yn;
        }
        lam[j] = rq;
      }
#undef AT
    }
    __syncthreads();
  }
  stamp(prof, 4);
  // modified Gram-Schmidt among close eigenvalues (twice)
  auto csum = [&](double v) {
    v = wsum(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    const double s = wsum(red[lane]);
    __syncthreads();
    return s;
  };
  for (int j = 1; j < m; ++j) {
    int i0 = j;
    while (i0 > 0 && lam[i0 - 1] - lam[i0] <= 1e-9) --i0;
    if (i0 == j) continue;
    for (int pass = 0; pass < 2; ++pass) {
      for (int i = i0; i < j; ++i) {
        double s = 0.0;
        for (int r = tid; r < n; r += kDT) s = fma(Y[r * m + i], Y[r * m + j], s);
        s = csum(s);
        for (int r = tid; r < n; r += kDT) Y[r * m + j] -= s * Y[r * m + i];
        __syncthreads();
      }
      double s = 0.0;
      for (int r = tid; r < n; r += kDT) s = fma(Y[r * m + j], Y[r * m + j], s);
      s = 1.0 / sqrt(csum(s));
      for (int r = tid; r < n; r += kDT) Y[r * m + j] *= s;
      __syncthreads();
    }
  }
  stamp(prof, 5);
  // ---- 4. back-transformation, a warp per vector (Yt: [m][n] copy, conflict-free lanes)
  double* Yt = dl;  // the inverse-iteration arrays are free now (n m <= 4 n R + ... checked on the host)
  for (int e = tid; e < n * m; e += kDT) {
    const int jj = e / n, r = e - jj * n;
    Yt[e] = Y[r * m + jj];
  }
  __syncthreads();
  // reflector rows staged in shared memory in chunks of CH (the workspace past Y and Yt, minus
  // room for the blocks' T factors), applied in blocks of kWB as compact-WY products
  // H_k0 .. H_k0+b-1 = I - V T V^T (T upper triangular, LAPACK dlarft forward / columnwise):
  // one warp-wide reduction per block instead of per reflector
  constexpr int kWB = 8;
  double* Hs = Yt + (size_t)n * m;
  // per chunk row: n doubles of Hs, 1 beta, kWB^2 / kWB = 8 of T (+ one spare block)
  const int CH = max(kWB, min(n, (int)((wsz - 2 * n * m - 64) / (n + 9)) / kWB * kWB));
  double* Tb = Hs + (size_t)CH * n;          // T factors of the chunk's blocks (kWB x kWB each)
  double* bet = Tb + (size_t)(CH / kWB + 1) * kWB * kWB;  // the chunk's betas
  for (int k1 = n - 2; k1 > 0; k1 -= CH) {  // rows [k0, k1) of H, applied last to first
    const int k0 = max(0, k1 - CH);
    for (int r = tid; r < k1 - k0; r += kDT) {
      const int k = k0 + r;
      bet[r] = betag ? betag[k] : Hg[(int64_t)k * n + k];
    }
    for (int e = tid; e < (k1 - k0) * n; e += kDT) {
      const int r = e / n, c = e - r * n;  // reflector k = k0 + r lives on entries c > k
      Hs[e] = c > k0 + r ? Hg[(int64_t)k0 * n + e] : 0.0;
    }
    __syncthreads();
    // T factors: blocks [kb0, kb0 + b) from the chunk's top down; dots of the block's columns
    const int nblk = (k1 - k0 + kWB - 1) / kWB;
    for (int q = warp; q < nblk * kWB * kWB; q += kDW) {
      const int blk = q / (kWB * kWB), ij = q - blk * (kWB * kWB), a = ij / kWB, c = ij - a * kWB;
      const int kb1 = k1 - blk * kWB, kb0 = max(k0, kb1 - kWB);
      const int bsz = kb1 - kb0;
      double dotv = 0.0;
      if (a < c && c < bsz) {
        const double* va = Hs + (size_t)(kb0 + a - k0) * n;
        const double* vc = Hs + (size_t)(kb0 + c - k0) * n;
        for (int r = lane; r < n; r += 32) dotv = fma(va[r], vc[r], dotv);
        dotv = wsum(dotv);
      }
      if (lane == 0) Tb[blk * kWB * kWB + ij] = dotv;  // V_a . V_c above the diagonal, for now
    }
    __syncthreads();
    for (int blk = tid; blk < nblk; blk += kDT) {  // T(0:i, i) = -beta_i T(0:i, 0:i) (V(:, 0:i)^T v_i)
      const int kb1 = k1 - blk * kWB, kb0 = max(k0, kb1 - kWB);
      const int bsz = kb1 - kb0;
      double* T = Tb + blk * kWB * kWB;
      // fully unrolled so column i's dots sit in registers (r1: a dynamically indexed 8 x 8 local
      // array, i.e. local-memory round trips on the chain)
#pragma unroll
      for (int i = 0; i < kWB; ++i) {
        double dcol[kWB];  // V_l . V_i, l < i (column i above the diagonal, overwritten below)
#pragma unroll
        for (int l = 0; l < kWB; ++l) dcol[l] = l < i ? T[l * kWB + i] : 0.0;
        const double bi = i < bsz ? bet[kb0 + i - k0] : 0.0;
#pragma unroll
        for (int a = 0; a < kWB; ++a) {
          if (a < i) {
            double t = 0.0;
#pragma unroll
            for (int l = 0; l < kWB; ++l)
              if (l >= a && l < i) t = fma(T[a * kWB + l], dcol[l], t);
            T[a * kWB + i] = -bi * t;
          }
        }
        T[i * kWB + i] = bi;
#pragma unroll
        for (int a = 0; a < kWB; ++a)
          if (a > i) T[a * kWB + i] = 0.0;
      }
    }
    __syncthreads();
    for (int jj = warp; jj < m; jj += kDW) {
      double* y = Yt + (size_t)jj * n;
      for (int blk = 0; blk < nblk; ++blk) {  // the chunk's last block first
        const int kb1 = k1 - blk * kWB, kb0 = max(k0, kb1 - kWB);
        const double* V = Hs + (size_t)(kb0 - k0) * n;
        const double* T = Tb + blk * kWB * kWB;
        double w[kWB];
#pragma unroll
        for (int l = 0; l < kWB; ++l) w[l] = 0.0;
        for (int r = kb0 + 1 + lane; r < n; r += 32) {
          const double yr = y[r];
#pragma unroll
          for (int l = 0; l < kWB; ++l) w[l] = fma(V[(size_t)l * n + r], yr, w[l]);  // rows past the block: zero T
        }
#pragma unroll
        for (int l = 0; l < kWB; ++l) w[l] = wsum(w[l]);
        double w2[kWB];
#pragma unroll
        for (int a = 0; a < kWB; ++a) {
          double t = 0.0;
#pragma unroll
          for (int c = 0; c < kWB; ++c) t = fma(T[a * kWB + c], w[c], t);
          w2[a] = t;
        }
        for (int r = kb0 + 1 + lane; r < n; r += 32) {
          double yr = y[r];
#pragma unroll
          for (int l = 0; l < kWB; ++l) yr = fma(-V[(size_t)l * n + r], w2[l], yr);
          y[r] = yr;
        }
        __syncwarp();
      }
    }
    __syncthreads();
  }
  stamp(prof, 6);
  for (int e = tid; e < n * m; e += kDT) {
    const int r = e / m, jj = e - r * m;
    Vout[e] = Yt[(size_t)jj * n + r];
  }
  for (int jj = tid; jj < m; jj += kDT) theta_out[jj] = lam[jj] * tn;
  if (tid < 8) info_out[tid] = tid == 0 || tid == 1 ? 1 : 0;  // converged (direct method), 1 "iteration"
  if (tid == 0) {
    double* dv = reinterpret_cast<double*>(info_out + 8);
    dv[0] = -1.0;  // no Lanczos / filter-bound estimates (eig_check keeps the slot's)
    dv[1] = -1.0;
  }
  stamp(prof, 7);
}

__global__ void __launch_bounds__(kDT, 1) k_eig_direct(DirArgs p) {
  extern __shared__ double sm[];
  __shared__ double npart[kDW], kpart[kDW];
  __shared__ double lam[256];
  __shared__ double red[kDW];
  const int n = p.n, m = p.m, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // layout: ub[2][n] | pr[n] | uv[n] | sa[n] | se[n] | te2[n] | pb[1024] (product partials) | L (packed; later the workspace)
  double* ub = sm;
  double* pr = ub + 2 * n;
  double* uv = pr + n;  // u of the current step (u1 at k1)
  double* sa = uv + n;
  double* se = sa + n;
  double* te2 = se + n;
  double* pb = te2 + n;
  double* L = pb + 1024;
  const int wsz = p.ws - 7 * n - 1024;  // doubles from L on
  stamp(p.prof, 0);
  for (int i = warp; i < n; i += kDW)
    for (int j = lane; j <= i; j += 32) L[pidx(i, j)] = p.S[(int64_t)i * p.lds + j];
  __syncthreads();
  stamp(p.prof, 1);
  if (n >= 3) {  // first column (k = 0) and its norm
    double ss = 0.0;
    for (int i = 1 + warp; i < n; i += kDW) {
      if (lane == 0) {
        const double x = L[pidx(i, 0)];
        ub[i] = x;
        ss += x * x;
      }
    }
    if (lane == 0) npart[warp] = ss;
  }
  __syncthreads();
  // ---- 1. tridiagonalisation.  Per column k (active indices k1 = k + 1 .. n - 1), three phases
  // and three block barriers; x = S[k1.., k] (the column, kept in ub by the previous step):
  //   P  p~ = S_sub x: lanes = rows (32-row blocks), warps = (row block, column segment), partial
  //      sums per segment (no scalar is needed: S u = S x - alpha S e_k1 is fixed up in R)
  //   R  threads = rows: the reflector (alpha, beta, u), p = beta (p~ - alpha S[:, k1]), K partials
  //   U  S_sub -= u q^T + q u^T, q = p - K u (lanes = columns); the owner of column k1 emits the
  //      next step's x and its norm
  __shared__ double scal[2];
  for (int k = 0; k < n - 2; ++k) {
    const double* x = ub + (k & 1) * n;
    double* xn = ub + ((k + 1) & 1) * n;
    const int k1 = k + 1, na = n - k1;
    const int nrb = (na + 31) >> 5;
    // column segments per row block: a power of two, <= 32 / nrb warps in all, and >= ~16 columns
    // each (short steps use few warps: the per-warp setup would dominate)
    int lg = nrb == 1 ? 5 : (nrb == 2 ? 4 : (nrb <= 4 ? 3 : 2));
    while (lg > 0 && (na >> lg) < 16) --lg;
    const int nseg = 1 << lg;
    {  // P
      const int SL = (na + nseg - 1) >> lg;
      const int rbk = warp >> lg, sg = warp & (nseg - 1);
      if (rbk < nrb) {
        const int i0 = k1 + 32 * rbk + lane;
        const int i = min(i0, n - 1);  // lanes past the last row read row n - 1, discarded
        const int ti = (i * (i + 1)) / 2;
        const int jb = k1 + sg * SL, je = min(n, jb + SL);
        const int rlo = k1 + 32 * rbk;
        double acc0 = 0.0, acc1 = 0.0;
        int j = jb;
        const int e1 = min(je, rlo);  // row part: j < rlo <= i
        for (; j + 1 < e1; j += 2) {
          const double2 xx = make_double2(x[j], x[j + 1]);
          acc0 = fma(L[ti + j], xx.x, acc0);
          acc1 = fma(L[ti + j + 1], xx.y, acc1);
        }
        for (; j < e1; ++j) acc0 = fma(L[ti + j], x[j], acc0);
        const int e2 = min(je, rlo + 32);  // the diagonal band
        for (; j < e2; ++j) acc0 = fma(j <= i ? L[ti + j] : L[(j * (j + 1)) / 2 + i], x[j], acc0);
        int tj = (j * (j + 1)) / 2;  // column part: j > i
        for (; j + 1 < je; j += 2) {
          const int tj1 = tj + j + 1;
          acc0 = fma(L[tj + i], x[j], acc0);
          acc1 = fma(L[tj1 + i], x[j + 1], acc1);
          tj = tj1 + j + 2;
        }
        for (; j < je; ++j) {
          acc0 = fma(L[tj + i], x[j], acc0);
          tj += j + 1;
        }
        if (i0 < n) pb[sg * (32 * nrb) + (i0 - k1)] = acc0 + acc1;
      }
    }
    __syncthreads();
    if (warp < nrb) {  // R
      const double nx2 = wsum(npart[lane]);
      const double x0 = x[k1];
      const double nx = sqrt(nx2);
      const double alpha = x0 >= 0 ? -nx : nx;
      const double uu = 2.0 * (nx2 - alpha * x0);
      const double beta = uu > 0 ? 2.0 / uu : 0.0;
      const double u1 = x0 - alpha;
      const int i = k1 + tid;
      double kp = 0.0;
      if (i < n) {
        double s2 = 0.0;
        for (int g = 0; g < nseg; ++g) s2 += pb[g * (32 * nrb) + tid];
        const double pi = beta * fma(-alpha, L[pidx(i, k1)], s2);
        const double ui = i == k1 ? u1 : x[i];
        pr[i] = pi;
        uv[i] = ui;
        kp = pi * ui;
        p.H[(int64_t)k * n + i] = ui;
      }
      kp = wsum(kp);
      if (lane == 0) kpart[warp] = kp;
      if (tid == 0) {
        scal[0] = beta;
        scal[1] = u1;
        sa[k] = L[pidx(k, k)];
        se[k] = alpha;
        p.H[(int64_t)k * n + k] = beta;
      }
    } else if (lane == 0) {
      kpart[warp] = 0.0;
    }
    __syncthreads();
    {  // U: lanes = rows i (32-row blocks); the (row block, j <= i) pairs of the lower triangle
       // are split evenly over the warps (block rbk holds 32 (rbk + 1) columns of pairs)
      const double K = 0.5 * scal[0] * wsum(kpart[lane]);
      const int C = 16 * nrb * (nrb + 1);            // total (block, column) pairs
      const int WU = max(1, min(kDW, C >> 4));        // >= 16 columns of pairs per warp
      const int c0 = warp < WU ? (warp * C) / WU : C, c1 = warp < WU ? ((warp + 1) * C) / WU : C;
      double ss = 0.0;
      int rbk = 0;
      while (16 * (rbk + 1) * (rbk + 2) <= c0) ++rbk;  // block holding pair c0
      for (int c = c0; c < c1; ++rbk) {
        const int cb = 16 * rbk * (rbk + 1);          // first pair of block rbk
        const int rlo = k1 + 32 * rbk;
        const int jb = k1 + (c - cb), je = min(k1 + (min(c1, cb + 32 * (rbk + 1)) - cb), n);
        c = min(c1, cb + 32 * (rbk + 1));
        const int i0 = rlo + lane;
        const bool iv = i0 < n;
        const int i = min(i0, n - 1);
        const int ti = (i * (i + 1)) / 2;
        const double ui = uv[i];
        const double qi = fma(-K, ui, pr[i]);
        int j = jb;
        if (j == k1 && j < je) {  // column k1 below the diagonal: the next step's x
          const double uj = uv[j], qj = fma(-K, uj, pr[j]);
          const double v = fma(-ui, qj, fma(-qi, uj, L[ti + j]));
          if (iv) {
            L[ti + j] = v;
            if (i > k1) {
              xn[i] = v;
              ss = fma(v, v, ss);
            }
          }
          ++j;
        }
        const int e1 = min(je, rlo);  // j < rlo <= i: every valid lane
        for (; j + 1 < e1; j += 2) {
          const double2 u2 = make_double2(uv[j], uv[j + 1]);
          const double2 p2 = make_double2(pr[j], pr[j + 1]);
          const double q0 = fma(-K, u2.x, p2.x), q1 = fma(-K, u2.y, p2.y);
          const double v0 = fma(-ui, q0, fma(-qi, u2.x, L[ti + j]));
          const double v1 = fma(-ui, q1, fma(-qi, u2.y, L[ti + j + 1]));
          if (iv) {
            L[ti + j] = v0;
            L[ti + j + 1] = v1;
          }
        }
        for (; j < je; ++j) {  // the rest, including the diagonal band (j <= i per lane)
          const double uj = uv[j], qj = fma(-K, uj, pr[j]);
          if (iv && j <= i) L[ti + j] = fma(-ui, qj, fma(-qi, uj, L[ti + j]));
        }
      }
      ss = wsum(ss);
      if (lane == 0) npart[warp] = ss;
    }
    __syncthreads();
  }
  if (tid == 0) {
    for (int i = max(0, n - 2); i < n; ++i) sa[i] = L[pidx(i, i)];
    if (n >= 2) se[n - 2] = L[pidx(n - 1, n - 2)];
    se[n - 1] = 0.0;
  }
  for (int k = max(0, n - 2) + tid / 256; k < n; k += kDT / 256)  // no reflector for the last two columns
    for (int i = tid % 256; i < n; i += 256) p.H[(int64_t)k * n + i] = 0.0;
  __syncthreads();
  stamp(p.prof, 2);
  eig_tail(n, m, sa, se, te2, L, wsz, lam, red, p.H, nullptr, p.V, p.theta, p.info, p.prof);
}


// ---- the tiled one-CTA tridiagonalisation (n <= 208; r2 default for the direct solver) ----
// S (both triangles' values: the lower triangle's tiles; diagonal tiles full) as 16 x 16 fp64
// tiles in shared memory, element (r, c) of a tile at c * 16 + (r ^ c): a half-warp reading a
// tile column (lanes = rows) or a tile row (lanes = columns) touches 16 distinct bank pairs, so
// both the row and the transposed column sweeps are conflict-free (the packed triangle of
// k_eig_direct read rows at lane strides of ~i doubles).  Per column k, two block barriers:
//   phase 1 (threads = rows i > k): the reflector of x_k = A[k+1.., k] (alpha, beta, u), from
//     the partial sums s = A x_k of the previous pass: p = beta (s - alpha A e_k1), K = beta^2 / 2
//     u^T A u with u^T A u = x^T A x - 2 alpha s_k1 + alpha^2 A_k1k1 (x^T A x from per-warp tile
//     partials), q = p - K u, and the next column x_{k+1} = (A - u q^T - q u^T)[k+2.., k+1];
//   phase 2 (warps = tiles of the active trailing block): A -= u q^T + q u^T and, in the same
//     sweep, the partial sums of A_new x_{k+1} (row sums, then the transposed column sums of
//     off-diagonal tiles) and x^T A_new x.
// One read + write of the trailing matrix per column (k_eig_direct: a product read and an
// update read + write).  Symmetric matrix; the reflectors are LAPACK dsytd2's (lower).
constexpr int kTB = 16;           // tile edge
constexpr int kTNB = 13;          // tile blocks: n <= 208
constexpr int kTN = kTB * kTNB;   // 208

__device__ __forceinline__ int toff(int I, int J) { return ((I * (I + 1)) / 2 + J) * (kTB * kTB); }  // I >= J
__device__ __forceinline__ int tel(int r, int c) { return c * kTB + (r ^ c); }
__device__ __forceinline__ int tat(int i, int j) {  // element (i, j), any order
  const int a = max(i, j), b = min(i, j);
  return toff(a >> 4, b >> 4) + tel(a & 15, b & 15);
}

// phase 2 over the tiles (I, J), B0 <= J <= I < nb: update with (u, q), partial sums of A x
// into pb[(I nb + J) 16 + r] (row part of tile (I, J)) and pb[(J nb + I) 16 + c] (column part)
__device__ __forceinline__ void tri_pass(double* T, double* pb, const double2* uq, const double* x, int nb, int B0,
                                         int warp, int lane, double* xpart) {
  // uq[i] = (u_i, q_i).  Shared-memory operands are staged in registers four columns at a time
  // before the tile's stores (the compiler cannot move loads across stores into the same array:
  // a load -> fma -> store chain per element was ~2.5x slower)
  const int mb = nb - B0;
  const int nt = mb * (mb + 1) / 2;
  const int r = lane & 15, h = lane >> 4;
  double xs = 0.0;
  for (int t = warp; t < nt; t += kDW) {
    int a = 0;
    while ((a + 1) * (a + 2) / 2 <= t) ++a;
    const int I = B0 + a, J = B0 + (t - a * (a + 1) / 2);
    double* Tt = T + toff(I, J);
    const double2 wr = uq[I * kTB + r];
    const double xr = x[I * kTB + r];
    double racc0 = 0.0, racc1 = 0.0;
#pragma unroll
    for (int c4 = 0; c4 < 8; c4 += 4) {
      double av[4], xc[4];
      double2 wc[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = h * 8 + c4 + j;
        av[j] = Tt[c * kTB + (r ^ c)];
        wc[j] = uq[J * kTB + c];
        xc[j] = x[J * kTB + c];
      }
      if (I != J) {
#pragma unroll
        for (int j = 0; j < 4; ++j) av[j] = fma(-wr.x, wc[j].y, fma(-wr.y, wc[j].x, av[j]));
      } else {  // diagonal tile, both triangles: a symmetric update formula keeps it exactly symmetric
#pragma unroll
        for (int j = 0; j < 4; ++j) av[j] = av[j] - __dadd_rn(__dmul_rn(wr.x, wc[j].y), __dmul_rn(wr.y, wc[j].x));
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = h * 8 + c4 + j;
        Tt[c * kTB + (r ^ c)] = av[j];
      }
      racc0 = fma(av[0], xc[0], racc0);
      racc1 = fma(av[1], xc[1], racc1);
      racc0 = fma(av[2], xc[2], racc0);
      racc1 = fma(av[3], xc[3], racc1);
    }
    double racc = racc0 + racc1;
    racc += __shfl_xor_sync(0xffffffffu, racc, 16);
    if (h == 0) {
      pb[(I * nb + J) * kTB + r] = racc;
      xs = fma(I != J ? 2.0 * xr : xr, racc, xs);
    }
    if (I != J) {  // column sums of the updated tile: lanes = columns, rows split by half-warp
      __syncwarp();
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int r4 = 0; r4 < 8; r4 += 4) {
        double av[4], xv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r2 = h * 8 + r4 + j;
          av[j] = Tt[r * kTB + (r2 ^ r)];
          xv[j] = x[I * kTB + r2];
        }
        c0 = fma(av[0], xv[0], c0);
        c1 = fma(av[1], xv[1], c1);
        c0 = fma(av[2], xv[2], c0);
        c1 = fma(av[3], xv[3], c1);
      }
      double cacc = c0 + c1;
      cacc += __shfl_xor_sync(0xffffffffu, cacc, 16);
      if (h == 0) pb[(J * nb + I) * kTB + r] = cacc;
    }
  }
  xs = wsum(xs);
  if (lane == 0) xpart[warp] = xs;
}

__global__ void __launch_bounds__(kDT, 1) k_eig_direct_t(DirArgs p) {
  extern __shared__ double sm[];
  __shared__ double npart[2][kDW], xpart[kDW];
  __shared__ double lam[256];
  __shared__ double red[kDW];
  const int n = p.n, m = p.m, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = (n + kTB - 1) / kTB;
  // layout: sa | se | te2 | u | q | x[2] (kTN each) | pb (nb nb 16) | tiles; from pb on: the tail's workspace
  double* sa = sm;
  double* se = sa + kTN;
  double* te2 = se + kTN;
  double2* uq = reinterpret_cast<double2*>(te2 + kTN);  // (u_i, q_i) interleaved
  double* xb = te2 + 3 * kTN;
  double* pb = xb + 2 * kTN;
  double* T = pb + nb * nb * kTB;
  const int wsz = p.ws - 7 * kTN;
  stamp(p.prof, 0);
  for (int e = tid; e < 4 * kTN; e += kDT) te2[kTN + e] = 0.0;  // uq, x[0], x[1]
  const int ntile = nb * (nb + 1) / 2;
  for (int e = tid; e < ntile * kTB * kTB; e += kDT) {
    const int t = e >> 8, w = e & 255;
    int I = 0;
    while ((I + 1) * (I + 2) / 2 <= t) ++I;
    const int J = t - I * (I + 1) / 2;
    const int c = w >> 4, r = (w & 15) ^ c;
    const int i = I * kTB + r, j = J * kTB + c;
    double v = 0.0;
    if (i < n && j < n) v = i >= j ? p.S[(int64_t)i * p.lds + j] : p.S[(int64_t)j * p.lds + i];
    T[e] = v;
  }
  __syncthreads();
  stamp(p.prof, 1);
  {  // x_0 = A[1.., 0] and its norm
    double ss = 0.0;
    for (int i = tid; i < n; i += kDT)
      if (i >= 1) {
        const double v = T[tat(i, 0)];
        xb[i] = v;
        ss = fma(v, v, ss);
      }
    ss = wsum(ss);
    if (lane == 0) npart[0][warp] = ss;
  }
  __syncthreads();
  tri_pass(T, pb, uq, xb, nb, 0, warp, lane, xpart);  // u = q = 0: the product A x_0 only
  __syncthreads();
  long long cyc[4] = {0, 0, 0, 0};  // TUCKER_EIG_PROF: thread 0's cycles in phase 1 / barrier / phase 2 / barrier
  const bool pr0 = p.prof != nullptr && tid == 0;
  const int dbg = p.dbg;
  for (int k = 0; k < n - 2; ++k) {
    long long c0 = pr0 ? clock64() : 0;
    const int k1 = k + 1;
    const double* xc = xb + (k & 1) * kTN;
    double* xn = xb + ((k + 1) & 1) * kTN;
    const int bprev = k >> 4;  // first tile block of the previous pass
    const int nr = n - k;      // rows k .. n - 1
    if (warp < (nr + 31) >> 5 && !(dbg & 2)) {
      const double nx2 = wsum(npart[k & 1][lane]);
      const double xax = wsum(xpart[lane]);
      const double x0 = xc[k1];
      const double nx = sqrt(nx2);
      const double alpha = x0 >= 0 ? -nx : nx;
      const double uu = 2.0 * (nx2 - alpha * x0);
      const double beta = uu > 0 ? 2.0 / uu : 0.0;
      const double u1 = x0 - alpha;
      double sk1 = 0.0;
      {
        const double* pr = pb + ((k1 >> 4) * nb) * kTB + (k1 & 15);
        for (int b = bprev; b < nb; ++b) sk1 += pr[b * kTB];
      }
      const double a11 = T[tat(k1, k1)];
      const double uau = fma(alpha * alpha, a11, fma(-2.0 * alpha, sk1, xax));
      const double K = 0.5 * beta * beta * uau;
      const double q1 = fma(-K, u1, beta * fma(-alpha, a11, sk1));
      const int i = k + tid;
      double ss = 0.0;
      if (i == k) {
        uq[k] = make_double2(0.0, 0.0);
        xn[k] = 0.0;
        sa[k] = T[tat(k, k)];
        se[k] = alpha;
        p.H[(int64_t)k * n + k] = beta;
      } else if (i < n) {
        double si = 0.0;
        const double* pr = pb + ((i >> 4) * nb) * kTB + (i & 15);
        for (int b = bprev; b < nb; ++b) si += pr[b * kTB];
        const double ai = T[tat(i, k1)];
        const double pi = beta * fma(-alpha, ai, si);
        const double ui = i == k1 ? u1 : xc[i];
        const double qi = fma(-K, ui, pi);
        uq[i] = make_double2(ui, qi);
        const double xv = i == k1 ? 0.0 : fma(-ui, q1, fma(-qi, u1, ai));
        xn[i] = xv;
        ss = xv * xv;
        p.H[(int64_t)k * n + i] = ui;
      }
      ss = wsum(ss);
      if (lane == 0) npart[(k + 1) & 1][warp] = ss;
    } else if (lane == 0) {
      npart[(k + 1) & 1][warp] = 0.0;
    }
    long long c1 = pr0 ? clock64() : 0;
    __syncthreads();
    long long c2 = pr0 ? clock64() : 0;
    if (!(dbg & 1)) tri_pass(T, pb, uq, xn, nb, k1 >> 4, warp, lane, xpart);
    long long c3 = pr0 ? clock64() : 0;
    __syncthreads();
    if (pr0) {
      const long long c4 = clock64();
      cyc[0] += c1 - c0;
      cyc[1] += c2 - c1;
      cyc[2] += c3 - c2;
      cyc[3] += c4 - c3;
    }
  }
  if (pr0)
    for (int i = 0; i < 4; ++i) p.prof[8 + i] = (unsigned long long)cyc[i];
  if (tid == 0) {
    for (int i = max(0, n - 2); i < n; ++i) sa[i] = T[tat(i, i)];
    if (n >= 2) se[n - 2] = T[tat(n - 1, n - 2)];
    se[n - 1] = 0.0;
  }
  for (int k = max(0, n - 2) + tid / 256; k < n; k += kDT / 256)  // no reflector for the last two columns
    for (int i = tid % 256; i < n; i += 256) p.H[(int64_t)k * n + i] = 0.0;
  __syncthreads();
  stamp(p.prof, 2);
  eig_tail(n, m, sa, se, te2, pb, wsz, lam, red, p.H, nullptr, p.V, p.theta, p.info, p.prof);
}
}  // namespace

// the 4-CTA cluster tridiagonalisation (k_tridiag: T = (a, e), reflectors in rows of H, beta)
// followed by the one-CTA phases 2-4 (TUCKER_EIG_HYBRID=1, d <= 256)
__global__ void __launch_bounds__(kDT, 1) k_tri_tail(const double* __restrict__ a, const double* __restrict__ e, int n,
                                                   int m, int ws, const double* __restrict__ H,
                                                   const double* __restrict__ beta, double* V, double* theta,
                                                   int* info) {
  extern __shared__ double sm[];
  __shared__ double lam[256];
  __shared__ double red[kDW];
  double* sa = sm;
  double* se = sa + n;
  double* te2 = se + n;
  double* L = te2 + n;
  for (int i = threadIdx.x; i < n; i += kDT) {
    sa[i] = a[i];
    se[i] = i < n - 1 ? e[i] : 0.0;
  }
  __syncthreads();
  eig_tail(n, m, sa, se, te2, L, ws - 3 * n, lam, red, H, beta, V, theta, info);
}

// shared memory (doubles) k_eig_direct needs for (n, m); 0: does not fit
size_t eig_direct_ws(int n, int m) {
  if (n < 3 || n > 32 * kDJ || m < 1 || m > n || m > 256) return 0;
  const size_t np = (size_t)n * (n + 1) / 2;  // packed triangle
  // workspace from L on: Y (n m) + R (4 n + n / 8 + 1) with R >= 1, and the transposed copy (n m)
  size_t wsz = std::max(np, (size_t)n * m + (size_t)(4 * n + (n + 7) / 8 + 1) * std::min(m, 20));
  wsz = std::max(wsz, (size_t)2 * n * m + 16 * (size_t)n);  // + reflector chunks of >= 16 rows
  wsz = std::max(wsz, (size_t)2 * n * m + 8 * (size_t)(n + 9) + 64);  // >= one block of 8 rows with its T
  const size_t tot = 7 * (size_t)n + 1024 + wsz;
  return tot * sizeof(double) <= 218 * 1024 ? tot : 0;  // + ~6 KB static shared memory <= 227 KB
}

// shared memory (doubles) k_eig_direct_t needs for (n, m); 0: does not fit (n > 208 or the tail's workspace)
size_t eig_direct_t_ws(int n, int m) {
  if (n < 3 || n > kTN || m < 1 || m > n || m > 256) return 0;
  const size_t nb = (n + kTB - 1) / kTB;
  const size_t wk = nb * nb * kTB + nb * (nb + 1) / 2 * kTB * kTB;  // pb + tiles: the tail's workspace
  size_t need = std::max((size_t)n * m + (size_t)(4 * n + (n + 7) / 8 + 1) * std::min(m, 20),
                         (size_t)2 * n * m + 16 * (size_t)n);
  need = std::max(need, (size_t)2 * n * m + 8 * (size_t)(n + 9) + 64);
  if (need > wk) return 0;
  const size_t tot = 7 * (size_t)kTN + wk;
  return tot * sizeof(double) <= 220 * 1024 ? tot : 0;  // + ~4 KB static shared memory <= 227 KB
}

void eig_small(const double* S, int64_t n, int64_t lds, int m, double* V, double* theta, int* info, DBuf<double>& scratch,
               cudaStream_t st) {
  static const bool prof = std::getenv("TUCKER_EIG_PROF") != nullptr;  // tools: per-phase times on stderr
  static unsigned long long* prof_d = nullptr;
  if (prof && !prof_d) TK_CUDA(cudaMalloc(&prof_d, 16 * sizeof(unsigned long long)));
  const bool old_direct = std::getenv("TUCKER_EIG_DIRECT_OLD") != nullptr;  // tests, experiments
  const size_t wst = old_direct ? 0 : eig_direct_t_ws((int)n, m);
  if (wst && !std::getenv("TUCKER_EIG_CLUSTER")) {  // one CTA, tiled S in shared memory
    scratch.ensure((size_t)(n * n));
    DirArgs a;
    a.S = S;
    a.lds = lds;
    a.n = (int)n;
    a.m = m;
    a.ws = (int)wst;
    a.H = scratch.p;
    a.V = V;
    a.theta = theta;
    a.info = info;
    a.prof = prof ? prof_d : nullptr;
    a.dbg = std::getenv("TUCKER_EIG_DBG") ? std::atoi(std::getenv("TUCKER_EIG_DBG")) : 0;
    smem_optin((const void*)k_eig_direct_t, wst * sizeof(double));
    TK_LAUNCH(k_eig_direct_t, 1, kDT, wst * sizeof(double), st, a);
    if (g_eig_kernel_event) TK_CUDA(cudaEventRecord(g_eig_kernel_event, st));
    if (prof) {
      unsigned long long t[16];
      TK_CUDA(cudaStreamSynchronize(st));
      TK_CUDA(cudaMemcpy(t, prof_d, sizeof(t), cudaMemcpyDeviceToHost));
      std::fprintf(stderr, "eig_direct_t n=%d m=%d us: load %.1f tridiag %.1f bisect %.1f invit %.1f mgs %.1f back %.1f out %.1f total %.1f"
                   " | tridiag cycles/step: ph1 %.0f bar %.0f ph2 %.0f bar %.0f\n",
                   (int)n, m, (t[1] - t[0]) * 1e-3, (t[2] - t[1]) * 1e-3, (t[3] - t[2]) * 1e-3, (t[4] - t[3]) * 1e-3,
                   (t[5] - t[4]) * 1e-3, (t[6] - t[5]) * 1e-3, (t[7] - t[6]) * 1e-3, (t[7] - t[0]) * 1e-3,
                   (double)t[8] / (n - 2), (double)t[9] / (n - 2), (double)t[10] / (n - 2), (double)t[11] / (n - 2));
    }
    return;
  }
  if (n < 3 || n > kNMax || m < 1 || m > n) fail(TUCKER_E_ARG, "eig_small: 3 <= n <= 256, 1 <= m <= n");
  const size_t ws = eig_direct_ws((int)n, m);
  if (ws && !std::getenv("TUCKER_EIG_CLUSTER")) {  // one CTA, everything in shared memory
    scratch.ensure((size_t)(n * n));
    DirArgs a;
    a.S = S;
    a.lds = lds;
    a.n = (int)n;
    a.m = m;
    a.ws = (int)ws;
    a.H = scratch.p;
    a.V = V;
    a.theta = theta;
    a.info = info;
    a.prof = prof ? prof_d : nullptr;
    a.dbg = 0;
    smem_optin((const void*)k_eig_direct, ws * sizeof(double));
    TK_LAUNCH(k_eig_direct, 1, kDT, ws * sizeof(double), st, a);
    if (g_eig_kernel_event) TK_CUDA(cudaEventRecord(g_eig_kernel_event, st));
    if (prof) {
      unsigned long long t[8];
      TK_CUDA(cudaStreamSynchronize(st));
      TK_CUDA(cudaMemcpy(t, prof_d, sizeof(t), cudaMemcpyDeviceToHost));
      std::fprintf(stderr, "eig_direct n=%d m=%d us: load %.1f tridiag %.1f bisect %.1f invit %.1f mgs %.1f back %.1f out %.1f total %.1f\n",
                   (int)n, m, (t[1] - t[0]) * 1e-3, (t[2] - t[1]) * 1e-3, (t[3] - t[2]) * 1e-3, (t[4] - t[3]) * 1e-3,
                   (t[5] - t[4]) * 1e-3, (t[6] - t[5]) * 1e-3, (t[7] - t[6]) * 1e-3, (t[7] - t[0]) * 1e-3);
    }
    return;
  }
  scratch.ensure((size_t)(3 * n + n * n + (size_t)m * n + (size_t)m * 5 * n));
  const bool hybrid = std::getenv("TUCKER_EIG_HYBRID") != nullptr;
  double* a = scratch.p;
  double* e = a + n;
  double* beta = e + n;
  double* H = beta + n;
  double* Y = H + n * n;
  double* F = Y + (size_t)m * n;
  TriArgs p;
  p.S = S;
  p.lds = lds;
  p.n = (int)n;
  p.a = a;
  p.e = e;
  p.H = H;
  p.beta = beta;
  const size_t smem = (size_t)kRows * kNMax * sizeof(double);
  smem_optin((const void*)k_tridiag, smem);
  TK_LAUNCH(k_tridiag, kCl, kNT, smem, st, p);
  if (hybrid) {
    const size_t wsz = std::max<size_t>(std::max<size_t>((size_t)n * m + (size_t)(4 * n + (n + 7) / 8 + 1) * std::min(m, 20),
                                                         (size_t)2 * n * m + 16 * (size_t)n),
                                        (size_t)2 * n * m + 8 * (size_t)(n + 9) + 64);
    const size_t ws = 3 * (size_t)n + wsz;
    if (ws * sizeof(double) <= 218 * 1024) {
      smem_optin((const void*)k_tri_tail, ws * sizeof(double));
      TK_LAUNCH(k_tri_tail, 1, kDT, ws * sizeof(double), st, a, e, (int)n, m, (int)ws, H, beta, V, theta, info);
      return;
    }
  }
  TK_LAUNCH(k_tri_eig, 1, 256, 0, st, a, e, (int)n, H, beta, m, Y, F, V, theta, info);
}

}  // namespace tk
