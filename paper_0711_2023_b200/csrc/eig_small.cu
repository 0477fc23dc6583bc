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

}  // namespace

void eig_small(const double* S, int64_t n, int64_t lds, int m, double* V, double* theta, int* info, DBuf<double>& scratch,
               cudaStream_t st) {
  if (n < 3 || n > kNMax || m < 1 || m > n) fail(TUCKER_E_ARG, "eig_small: 3 <= n <= 256, 1 <= m <= n");
  scratch.ensure((size_t)(3 * n + n * n + (size_t)m * n + (size_t)m * 5 * n));
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
  TK_LAUNCH(k_tri_eig, 1, 256, 0, st, a, e, (int)n, H, beta, m, Y, F, V, theta, info);
}

}  // namespace tk
