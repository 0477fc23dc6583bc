// eig.cu -- post-processing of the eigensolver output (eig_fused.cu):
//   * CholQR2 of a tall fp64 block (the Y^T Y route, U = Y_(n) V Theta^{-1/2},
//     DESIGN.md reading A10), with a one-CTA Cholesky + triangular inverse;
//   * sign canonicalisation (largest |entry| positive, ties -> lowest index;
//     SPEC S:136, reading A3) and the fp32 conversion of the factor.
#include <algorithm>
#include <cmath>

#include "internal.cuh"

namespace tk {
namespace {

// ------------------------------------------------------- Cholesky / inverse --
// One CTA of 256 threads (8 warps).  G (k x k SPD) is equilibrated to unit
// diagonal (D G D, D = diag(G)^-1/2) and shifted by `shift` I, factored as
// R^T R (R upper) and inverted; Rinv = D R^{-1}, so Y Rinv has orthonormal
// columns when G = Y^T Y.  Both loops are right-looking with one barrier per
// step: the pivot row is cached in registers (lane owns columns lane + 32c)
// and every warp updates its own rows, so no long dependent chains.
// rj[idx] with a warp-uniform runtime idx, without a local-memory array
template <int NC>
__device__ __forceinline__ double pick(const double (&r)[NC], int idx) {
  double v = r[0];
#pragma unroll
  for (int c = 1; c < NC; ++c)
    if (idx == c) v = r[c];
  return v;
}

template <int NC>
__global__ void __launch_bounds__(256) k_chol_inv(const double* __restrict__ G, int k,
                                                  double* __restrict__ Rinv, double shift) {
  extern __shared__ double sm[];
  const int ld = k + 1;
  double* A = sm;           // k x ld : upper triangle -> R, then column-scaled R
  double* X = sm + k * ld;  // k x ld : R^{-1}
  __shared__ double dsc[kMaxBlock];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int nw = nt >> 5;
  for (int i = tid; i < k; i += nt) {
    const double g = G[i * k + i];
    dsc[i] = g > 0 ? 1.0 / sqrt(g) : 1.0;
  }
  __syncthreads();
  for (int r = warp; r < k; r += nw)
    for (int c = lane; c < k; c += 32) {
      A[r * ld + c] = G[r * k + c] * dsc[r] * dsc[c] + (r == c ? shift : 0.0);
      X[r * ld + c] = (r == c) ? 1.0 : 0.0;
    }
  __syncthreads();
  // ---- Cholesky: step j scales row j by 1/sqrt(pivot) and updates rows l > j
  double rj[NC];
  for (int j = 0; j < k; ++j) {
    if (j > 0 && warp == 0) {
      // publish the scaled row j-1 (every warp has read it during step j-1)
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int m = lane + 32 * c;
        if (m >= j - 1 && m < k) A[(j - 1) * ld + m] = rj[c];
      }
    }
    const double dj = A[j * ld + j];
    const double piv = sqrt(dj > 1e-12 ? dj : 1e-12);
    const double ipiv = 1.0 / piv;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int m = lane + 32 * c;
      rj[c] = (m > j && m < k) ? A[j * ld + m] * ipiv : (m == j ? piv : 0.0);
    }
    for (int l = j + 1 + warp; l < k; l += nw) {
      const double ajl = __shfl_sync(0xffffffffu, pick<NC>(rj, l >> 5), l & 31);
      double* al = A + l * ld;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int m = lane + 32 * c;
        if (m >= l && m < k) al[m] -= ajl * rj[c];
      }
    }
    __syncthreads();
  }
  if (warp == 0) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int m = lane + 32 * c;
      if (m >= k - 1 && m < k) A[(k - 1) * ld + m] = rj[c];
    }
  }
  __syncthreads();
  // ---- X = R^{-1}: back substitution in rank-1 form, X[i][:] -= (R[i][l]/R[l][l]) X[l][:]
  for (int i = warp; i < k; i += nw)
    for (int l = i + 1 + lane; l < k; l += 32) A[i * ld + l] = A[i * ld + l] / A[l * ld + l];
  __syncthreads();
  for (int l = k - 1; l > 0; --l) {
    double xl[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int j = lane + 32 * c;
      xl[c] = (j >= l && j < k) ? X[l * ld + j] : 0.0;
    }
    for (int i = warp; i < l; i += nw) {
      const double bil = A[i * ld + l];
      double* xi = X + i * ld;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int j = lane + 32 * c;
        if (j >= l && j < k) xi[j] -= bil * xl[c];
      }
    }
    __syncthreads();
  }
  for (int i = warp; i < k; i += nw) {
    const double s = dsc[i] / A[i * ld + i];
    for (int j = lane; j < k; j += 32) Rinv[i * k + j] = s * X[i * ld + j];
  }
}

void launch_chol_inv(const double* G, int k, double* Rinv, double shift, cudaStream_t st) {
  const size_t smem = (size_t)2 * k * (k + 1) * sizeof(double);
  const int nc = (k + 31) / 32;
  if (nc <= 1) TK_LAUNCH(k_chol_inv<1>, 1, 256, smem, st, G, k, Rinv, shift);
  else if (nc == 2) TK_LAUNCH(k_chol_inv<2>, 1, 256, smem, st, G, k, Rinv, shift);
  else if (nc == 3) TK_LAUNCH(k_chol_inv<3>, 1, 256, smem, st, G, k, Rinv, shift);
  else TK_LAUNCH(k_chol_inv<4>, 1, 256, smem, st, G, k, Rinv, shift);
}

__global__ void k_copy_cols(const double* __restrict__ src, int64_t lds, double* __restrict__ dst,
                            int64_t ldd, int64_t d, int ncol) {
  const int64_t n = d * ncol;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / ncol;
    const int c = (int)(e % ncol);
    dst[r * ldd + c] = src[r * lds + c];
  }
}

// sign canonicalisation (largest |entry| positive, ties -> lowest index)
// and fp32 conversion.  One CTA per column.
__global__ void k_canon_f32(const double* __restrict__ V, int64_t ldv, int64_t d, int J,
                            float* __restrict__ U) {
  __shared__ double bv[256];
  __shared__ int64_t bi[256];
  const int j = blockIdx.x;
  double best = -1.0;
  int64_t bidx = 0;
  for (int64_t r = threadIdx.x; r < d; r += blockDim.x) {
    const double a = fabs(V[r * ldv + j]);
    if (a > best) { best = a; bidx = r; }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = bidx;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const double o = bv[threadIdx.x + w];
      const int64_t oi = bi[threadIdx.x + w];
      if (o > bv[threadIdx.x] || (o == bv[threadIdx.x] && oi < bi[threadIdx.x])) {
        bv[threadIdx.x] = o;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  const double sgn = V[bi[0] * ldv + j] < 0 ? -1.0 : 1.0;
  for (int64_t r = threadIdx.x; r < d; r += blockDim.x) U[r * J + j] = (float)(sgn * V[r * ldv + j]);
}

inline int grid_for(int64_t n) {
  int64_t g = ceil_div(n, 256);
  if (g > 148 * 8) g = 148 * 8;
  return (int)(g < 1 ? 1 : g);
}

MatRef f64(const double* p, int64_t ld, bool trans = false) {
  MatRef r;
  r.t = Elt::F64;
  r.p = p;
  r.ld = ld;
  r.trans = trans;
  return r;
}


// dynamic smem opt-in for the Cholesky kernel (2 k (k + 1) doubles)
void chol_attr() {
  const size_t bytes = 2 * kMaxBlock * (kMaxBlock + 1) * sizeof(double);
  smem_optin((const void*)k_chol_inv<1>, bytes);
  smem_optin((const void*)k_chol_inv<2>, bytes);
  smem_optin((const void*)k_chol_inv<3>, bytes);
  smem_optin((const void*)k_chol_inv<4>, bytes);
}

// Q (d x k) <- Q R^{-1} twice (CholQR2)
void cholqr2_impl(double* Q, double* T, int64_t d, int k, EigWs& ws, cudaStream_t st) {
  chol_attr();
  for (int pass = 0; pass < 2; ++pass) {
    dgemm(k, k, d, 1.0, f64(Q, k, true), f64(Q, k), 0.0, ws.H.p, k, 0.0, nullptr, 0, ws.dense, st);
    launch_chol_inv(ws.H.p, k, ws.R.p, 0.0, st);
    dgemm(d, k, k, 1.0, f64(Q, k), f64(ws.R.p, k), 0.0, T, k, 0.0, nullptr, 0, ws.dense, st);
    TK_LAUNCH(k_copy_cols, grid_for(d * k), 256, 0, st, T, (int64_t)k, Q, (int64_t)k, d, k);
  }
}

}  // namespace

void cholqr2(double* V, int64_t ldv, int64_t d, int J, EigWs& ws, cudaStream_t st) {
  ws.cq.ensure((size_t)(d * J));
  ws.ct.ensure((size_t)(d * J));
  ws.H.ensure((size_t)J * J);
  ws.R.ensure((size_t)J * J);
  TK_LAUNCH(k_copy_cols, grid_for(d * J), 256, 0, st, V, ldv, ws.cq.p, (int64_t)J, d, J);
  cholqr2_impl(ws.cq.p, ws.ct.p, d, J, ws, st);
  TK_LAUNCH(k_copy_cols, grid_for(d * J), 256, 0, st, ws.cq.p, (int64_t)J, V, ldv, d, J);
}

void canon_to_f32(const double* V, int64_t ldv, int64_t d, int J, float* U, cudaStream_t st) {
  TK_LAUNCH(k_canon_f32, J, 256, 0, st, V, ldv, d, J, U);
}

}  // namespace tk
