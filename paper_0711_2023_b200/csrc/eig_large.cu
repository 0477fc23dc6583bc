// eig_large.cu -- J leading eigenvectors of a large symmetric PSD matrix (d > kFusedMaxD:
// MP's M_1, M_2 at config 5 are 50000 x 50000).  Fig. 7 "A <- J leading eigenvectors
// of M" (MATLAB eigs).
//
// The persistent solver (eig_fused.cu) keeps every CTA's rows of the Ritz block in
// shared memory, which caps d near 64 x #SMs.  This host-driven variant runs the same
// method -- Chebyshev-filtered block subspace iteration with locking, CholQR2 and a
// Rayleigh-Ritz step -- as a sequence of library kernels: the S Q products on the fp64
// GEMM (dense.cu), the k x k Rayleigh-Ritz problem on the one-CTA Jacobi of the fused
// solver (eig_unit), CholQR2 (eig.cu).  Converged leading Ritz pairs (residual
// ||S q - theta q|| <= tol theta_1) are locked; the filter then acts on the active
// block projected against them, so the outlier theta_1 never dominates a filtered block
// (the filter degree is capped so the block stays within CholQR2's reach).  One host
// synchronisation per outer iteration reads the Ritz values and residuals.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "internal.cuh"

namespace tk {
namespace {

__global__ void k_seed_large(double* __restrict__ Q, int64_t d, int k, const float* __restrict__ hint, int J,
                             uint64_t seed) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < d * k; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / k;
    const int c = (int)(e - r * k);
    double v;
    if (hint && c < J) {
      v = (double)hint[r * J + c];
    } else {
      uint64_t z = seed ^ ((uint64_t)r * 0x9E3779B97F4A7C15ull + (uint64_t)c * 0xBF58476D1CE4E5B9ull);
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      z ^= z >> 31;
      v = (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
    }
    Q[e] = v;
  }
}

// res[j] = ||SQ[:, j] - theta[j] Q[:, j]||^2 for j < n (one CTA per column, fixed order)
__global__ void k_col_residual(const double* __restrict__ SQ, const double* __restrict__ Q, int64_t d, int ld,
                               const double* __restrict__ theta, double* __restrict__ res) {
  __shared__ double red[256];
  const int j = blockIdx.x;
  const double t = theta[j];
  double s = 0.0;
  for (int64_t r = threadIdx.x; r < d; r += blockDim.x) {
    const double v = SQ[r * ld + j] - t * Q[r * ld + j];
    s = fma(v, v, s);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) res[j] = red[0];
}

// dst[:, c0 + c] = src[:, c] (d rows, n columns; row strides lds / ldd)
__global__ void k_copy_block(const double* __restrict__ src, int lds, double* __restrict__ dst, int ldd, int64_t d,
                             int c0, int n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < d * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / n;
    const int c = (int)(e - r * n);
    dst[r * ldd + c0 + c] = src[r * lds + c];
  }
}

// W[:, j] *= lambda_j^{-1/2} (k x k, row-major), 0 for lambda_j <= 0
__global__ void k_scale_rsqrt_cols(double* W, int k, const double* __restrict__ lam) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * k; e += gridDim.x * blockDim.x) {
    const double l = lam[e % k];
    W[e] *= l > 0 ? 1.0 / sqrt(l) : 0.0;
  }
}

inline unsigned grid_of(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 148 * 8)); }

MatRef f64m(const double* p, int64_t ld, bool trans = false) {
  MatRef r;
  r.t = Elt::F64;
  r.p = p;
  r.ld = ld;
  r.trans = trans;
  return r;
}

}  // namespace

bool eig_large(const double* S, int64_t d, int64_t ls, int J, EigSlot& slot, EigWs& ws, const EigOpts& o,
               double* out_V, double* theta_dev, int* info_dev, cudaStream_t st, const float* hint) {
  const int k = (int)std::min<int64_t>(kSmallMaxD, std::min<int64_t>(d, J + std::max(8, std::min(J, 10))));
  // blocks wider than the one-CTA Jacobi / CholQR (k > kMaxBlock): the Rayleigh-Ritz problem on the
  // direct dense solver (eig_small) and orthonormalisation by SVQB, Q <- Q W Lambda^{-1/2} with
  // Q^T Q = W Lambda W^T (twice; columns get re-mixed, which the next Rayleigh-Ritz step undoes)
  auto orth = [&](double* Qb, int kk) {
    if (kk <= kMaxBlock) {
      cholqr2(Qb, kk, d, kk, ws, st);
      return;
    }
    for (int pass = 0; pass < 2; ++pass) {
      dgemm(kk, kk, d, 1.0, f64m(Qb, kk, true), f64m(Qb, kk), 0.0, ws.sH.p, kk, 0.0, nullptr, 0, ws.dense, st);
      eig_small(ws.sH.p, kk, kk, kk, ws.sV.p, ws.sTh.p, ws.sInfo.p, ws.small, st);
      TK_LAUNCH(k_scale_rsqrt_cols, grid_of((int64_t)kk * kk), 256, 0, st, ws.sV.p, kk, ws.sTh.p);
      dgemm(d, kk, kk, 1.0, f64m(Qb, kk), f64m(ws.sV.p, kk), 0.0, ws.bT.p == Qb ? ws.bY1.p : ws.bT.p, kk, 0.0,
            nullptr, 0, ws.dense, st);
      double* out = ws.bT.p == Qb ? ws.bY1.p : ws.bT.p;
      TK_LAUNCH(k_copy_block, grid_of(d * kk), 256, 0, st, out, kk, Qb, kk, d, 0, kk);
    }
  };
  auto rr_eig = [&](int ka) {
    if (ka <= kMaxBlock) eig_unit(1, ws.sH.p, ka, ws.sV.p, ws.sTh.p, ws.sInfo.p, 40, 0.0, st);
    else eig_small(ws.sH.p, ka, ka, ka, ws.sV.p, ws.sTh.p, ws.sInfo.p, ws.small, st);
  };
  const double tol = o.tol;
  // work blocks d x k (fp64): L (locked, first nl columns valid), Q (active), SQ, Y0, Y1, T
  ws.bL.ensure((size_t)d * k);
  ws.bQ.ensure((size_t)d * k);
  ws.bSQ.ensure((size_t)d * k);
  ws.bY0.ensure((size_t)d * k);
  ws.bY1.ensure((size_t)d * k);
  ws.bT.ensure((size_t)d * k);
  ws.sH.ensure((size_t)k * k);
  ws.sV.ensure((size_t)k * k);
  ws.sC.ensure((size_t)k * k);
  ws.sTh.ensure((size_t)k);
  ws.sRes.ensure((size_t)k);
  ws.sInfo.ensure(16);
  double *L = ws.bL.p, *Q = ws.bQ.p, *SQ = ws.bSQ.p, *Y0 = ws.bY0.p, *Y1 = ws.bY1.p, *T = ws.bT.p;
  // start: the slot's basis of the last solve (same d, k), else the hint + pseudo-random columns
  const bool warm = slot.valid && slot.d == d && slot.k == k && slot.basis.n >= (size_t)d * k;
  if (warm) {
    TK_CUDA(cudaMemcpyAsync(Q, slot.basis.p, (size_t)d * k * sizeof(double), cudaMemcpyDeviceToDevice, st));
  } else {
    TK_LAUNCH(k_seed_large, grid_of(d * k), 256, 0, st, Q, d, k, hint, J, 0x1a29e5ull + (uint64_t)d * 131 + J);
  }
  orth(Q, k);

  int nl = 0;  // locked columns (leading Ritz pairs, descending)
  std::vector<double> th((size_t)k), res((size_t)k), lth;
  double theta1 = 0.0, lo = 0.0;
  int outer = 0, products = 0;
  bool converged = false, breakdown = false;
  const int max_outer = std::max(o.max_outer, 80);
  for (outer = 0; outer < max_outer; ++outer) {
    const int ka = k - nl;
    // Rayleigh-Ritz on the active block: SQ = S Q - L Theta_L L^T Q (= S Q: Q is orthogonal to L)
    dgemm(d, ka, d, 1.0, f64m(S, ls), f64m(Q, ka), 0.0, SQ, ka, 0.0, nullptr, 0, ws.dense, st);
    ++products;
    dgemm(ka, ka, d, 1.0, f64m(Q, ka, true), f64m(SQ, ka), 0.0, ws.sH.p, ka, 0.0, nullptr, 0, ws.dense, st);
    rr_eig(ka);
    dgemm(d, ka, ka, 1.0, f64m(Q, ka), f64m(ws.sV.p, ka), 0.0, T, ka, 0.0, nullptr, 0, ws.dense, st);
    std::swap(Q, T);
    dgemm(d, ka, ka, 1.0, f64m(SQ, ka), f64m(ws.sV.p, ka), 0.0, T, ka, 0.0, nullptr, 0, ws.dense, st);
    std::swap(SQ, T);
    TK_LAUNCH(k_col_residual, ka, 256, 0, st, SQ, Q, d, ka, ws.sTh.p, ws.sRes.p);
    int sw = 0;
    TK_CUDA(cudaMemcpyAsync(th.data(), ws.sTh.p, ka * sizeof(double), cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaMemcpyAsync(res.data(), ws.sRes.p, ka * sizeof(double), cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaMemcpyAsync(&sw, ws.sInfo.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaStreamSynchronize(st));
    if (sw < 0 || !std::isfinite(th[0])) {
      breakdown = true;
      break;
    }
    if (nl == 0) theta1 = th[0];
    // lock the converged leading Ritz pairs (contiguous from the top, up to J)
    int newl = 0;
    while (nl + newl < J && newl < ka && std::sqrt(res[newl]) <= tol * theta1) ++newl;
    if (newl > 0) {
      TK_LAUNCH(k_copy_block, grid_of(d * newl), 256, 0, st, Q, ka, L, k, d, nl, newl);
      for (int j = 0; j < newl; ++j) lth.push_back(th[j]);
      // the active block keeps its remaining columns
      const int kb = ka - newl;
      TK_LAUNCH(k_copy_block, grid_of(d * kb), 256, 0, st, Q + newl, ka, T, kb, d, 0, kb);
      std::swap(Q, T);
      nl += newl;
    }
    if (nl >= J) {
      converged = true;
      break;
    }
    const int kn = k - nl;  // active columns
    // filter interval [lo, cut]: the smallest active Ritz value bounds the unwanted part
    const double cut = th[ka - 1];
    const double top = th[newl];  // largest active Ritz value
    const double c = 0.5 * (cut + lo), e = 0.5 * (cut - lo);
    if (!(e > 0)) {
      breakdown = true;
      break;
    }
    // degree: amplification of the top active value over the cut <= ~1e5 (CholQR2 reach)
    const double rho_top = (top - c) / e;
    int m = 1;
    while (m < 12 && std::cosh((m + 1) * std::acosh(std::max(1.0, rho_top))) < 1e5) ++m;
    // Y_1 = (S Q - c Q) / e, Y_t = 2 (S Y_{t-1} - c Y_{t-1}) / e - Y_{t-2}, each projected against L
    auto project = [&](double* Y) {  // Y -= L (L^T Y)
      if (nl == 0) return;
      dgemm(nl, kn, d, 1.0, f64m(L, k, true), f64m(Y, kn), 0.0, ws.sC.p, kn, 0.0, nullptr, 0, ws.dense, st);
      dgemm(d, kn, nl, -1.0, f64m(L, k), f64m(ws.sC.p, kn), 1.0, Y, kn, 0.0, nullptr, 0, ws.dense, st);
    };
    const double* prev = Q;  // Y_0
    double* cur = Y0;
    dgemm4(d, kn, d, 1.0 / e, f64m(S, ls), f64m(prev, kn), 0.0, cur, kn, -c / e, prev, kn, 0.0, nullptr, 0, ws.dense,
           st);
    ++products;
    project(cur);
    double* spare = Y1;
    for (int t = 2; t <= m; ++t) {
      dgemm4(d, kn, d, 2.0 / e, f64m(S, ls), f64m(cur, kn), 0.0, spare, kn, -2.0 * c / e, cur, kn, -1.0, prev, kn,
             ws.dense, st);
      ++products;
      project(spare);
      double* freed = (prev == Q) ? T : const_cast<double*>(prev);
      prev = cur;
      cur = spare;
      spare = freed;
    }
    double* Yb = cur;
    // Q <- orthonormalised filtered block, orthogonal to L
    TK_LAUNCH(k_copy_block, grid_of(d * kn), 256, 0, st, Yb, kn, Q, kn, d, 0, kn);
    if (nl > 0) {
      dgemm(nl, kn, d, 1.0, f64m(L, k, true), f64m(Q, kn), 0.0, ws.sC.p, kn, 0.0, nullptr, 0, ws.dense, st);
      dgemm(d, kn, nl, -1.0, f64m(L, k), f64m(ws.sC.p, kn), 1.0, Q, kn, 0.0, nullptr, 0, ws.dense, st);
    }
    orth(Q, kn);
  }
  // result: V = [L | leading active Ritz vectors] (J columns, descending), theta
  std::vector<double> thJ((size_t)J);
  for (int j = 0; j < J; ++j) thJ[j] = j < nl ? lth[j] : (j - nl < (int)th.size() ? th[j - nl] : 0.0);
  if (nl > 0) TK_LAUNCH(k_copy_block, grid_of(d * nl), 256, 0, st, L, k, out_V, J, d, 0, std::min(nl, J));
  if (nl < J) TK_LAUNCH(k_copy_block, grid_of(d * (J - nl)), 256, 0, st, Q, k - nl, out_V, J, d, nl, J - nl);
  TK_CUDA(cudaMemcpyAsync(theta_dev, thJ.data(), J * sizeof(double), cudaMemcpyHostToDevice, st));
  // warm start for the next solve of this slot: [L | Q] as a d x k block
  slot.basis.ensure((size_t)d * k);
  if (nl > 0) TK_LAUNCH(k_copy_block, grid_of(d * nl), 256, 0, st, L, k, slot.basis.p, k, d, 0, nl);
  TK_LAUNCH(k_copy_block, grid_of(d * (k - nl)), 256, 0, st, Q, k - nl, slot.basis.p, k, d, nl, k - nl);
  slot.d = d;
  slot.k = k;
  slot.valid = converged && !breakdown;
  int info[8] = {converged ? 1 : 0, outer, products, 0, breakdown ? 1 : 0, 0, 0, 0};
  TK_CUDA(cudaMemcpyAsync(info_dev, info, sizeof(info), cudaMemcpyHostToDevice, st));
  TK_CUDA(cudaStreamSynchronize(st));  // host vectors go out of scope
  return converged;
}

}  // namespace tk
