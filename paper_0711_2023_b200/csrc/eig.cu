// eig.cu -- leading-J eigenvectors of a symmetric PSD fp64 matrix.
//
// Figs. 1-8 "A <- J leading eigenvectors of ..." (the paper calls MATLAB
// `eigs(M*M', J, 'lm')`, ARPACK; SURVEY reading A2 uses M itself).
// Method: block Chebyshev-filtered subspace
// iteration with block size k = J + p, CholQR2 orthonormalisation and a
// Rayleigh-Ritz step whose k x k eigenproblem is solved by a one-CTA cyclic
// Jacobi in shared memory (fp64).  Warm starts reuse the last Ritz basis of the
// same (algorithm, mode) slot.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "internal.cuh"

namespace tk {
namespace {

// ---------------------------------------------------------------- Jacobi ----
// One CTA of 1024 threads.  H (k x k, row-major) -> V (k x k) eigenvectors in
// columns and theta (k) eigenvalues, sorted descending.  k even, k <= kMaxBlock.
// Parallel cyclic Jacobi: each round applies k/2 disjoint rotations chosen by
// the circle-method tournament (k-1 rounds per sweep).  A round is three
// barrier-separated phases with contiguous, conflict-free shared-memory access:
//   1. warp t computes the rotation of slot t = (pos[t], pos[k-1-t]);
//   2. rows:    H <- J^T H and V^T <- J^T V^T   (lane = column);
//   3. columns: H <- H J                        (lane = row).
// Rows stay in place (indexed by matrix index), so no data moves between rounds.
// Rotations with |h_pq| <= tol sqrt(h_pp h_qq) are skipped; the sweep loop stops
// when a sweep makes no rotation or after max_sweeps (the caller's Ritz residuals
// decide convergence, so a capped solve only costs another outer iteration).
__global__ void __launch_bounds__(1024) k_jacobi(const double* __restrict__ Hin, int k,
                                                 double* __restrict__ Vout,
                                                 double* __restrict__ theta, int max_sweeps,
                                                 double tol, int* sweeps_out) {
  extern __shared__ double sm[];
  const int kin = k;
  k += (k & 1);             // odd k: one inert dummy index (zero coupling, sorts last)
  const int ld = k + 1;
  double* H = sm;           // k x ld
  double* W = sm + k * ld;  // k x ld : V^T (row i = eigenvector i)
  __shared__ double cs_c[kMaxBlock / 2], cs_s[kMaxBlock / 2];
  __shared__ int top[kMaxBlock / 2], bot[kMaxBlock / 2], act[kMaxBlock / 2];
  __shared__ int pos[kMaxBlock];
  __shared__ int order[kMaxBlock];
  __shared__ int bad;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int nw = nt >> 5;
  const int np = k / 2;
  for (int r = warp; r < k; r += nw)
    for (int c = lane; c < k; c += 32) {
      H[r * ld + c] = (r < kin && c < kin) ? 0.5 * (Hin[r * kin + c] + Hin[c * kin + r])
                                           : ((r == c) ? -1e300 : 0.0);
      W[r * ld + c] = (r == c) ? 1.0 : 0.0;
    }
  for (int i = tid; i < k; i += nt) pos[i] = i;
  __syncthreads();
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    int any_in_sweep = 0;
    for (int round = 0; round < k - 1; ++round) {
      // phase 1: rotations
      int my_act = 0;
      if (tid < np) {
        const int p = pos[tid], q = pos[k - 1 - tid];
        top[tid] = p;
        bot[tid] = q;
        const double app = H[p * ld + p], aqq = H[q * ld + q], apq = H[p * ld + q];
        double c = 1.0, s = 0.0;
        if (fabs(apq) > tol * sqrt(fabs(app * aqq)) && apq != 0.0) {
          const double tau = (aqq - app) / (2.0 * apq);
          const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          c = 1.0 / sqrt(1.0 + t * t);
          s = t * c;
          my_act = 1;
        }
        cs_c[tid] = c;
        cs_s[tid] = s;
        act[tid] = my_act;
      }
      const int any = __syncthreads_or(my_act);
      int nextpos = 0;
      if (tid < k) nextpos = (tid == 0) ? pos[0] : pos[tid == 1 ? k - 1 : tid - 1];
      if (any) {
        any_in_sweep = 1;
        // phase 2: rows p, q of H and of V^T  <-  J^T (rows)
        for (int P = warp; P < np; P += nw) {
          if (!act[P]) continue;
          const int p = top[P], q = bot[P];
          const double c = cs_c[P], s = cs_s[P];
          double* hp = H + p * ld;
          double* hq = H + q * ld;
          double* wp = W + p * ld;
          double* wq = W + q * ld;
          for (int j = lane; j < k; j += 32) {
            const double x = hp[j], y = hq[j];
            hp[j] = c * x - s * y;
            hq[j] = s * x + c * y;
            const double u = wp[j], v = wq[j];
            wp[j] = c * u - s * v;
            wq[j] = s * u + c * v;
          }
        }
        __syncthreads();
        // phase 3: columns p, q of H  <-  H J (lane = row)
        for (int P = warp; P < np; P += nw) {
          if (!act[P]) continue;
          const int p = top[P], q = bot[P];
          const double c = cs_c[P], s = cs_s[P];
          for (int i = lane; i < k; i += 32) {
            const double x = H[i * ld + p], y = H[i * ld + q];
            H[i * ld + p] = c * x - s * y;
            H[i * ld + q] = s * x + c * y;
          }
        }
        __syncthreads();
        // exact zero in the rotated 2x2 blocks
        if (tid < np && act[tid]) {
          H[top[tid] * ld + bot[tid]] = 0.0;
          H[bot[tid] * ld + top[tid]] = 0.0;
        }
      }
      if (tid < k) pos[tid] = nextpos;  // circle method: keep pos[0], rotate the rest
      __syncthreads();
    }
    if (!any_in_sweep) break;
  }
  // sort eigenvalues descending (stable by index)
  if (tid == 0) bad = 0;
  if (tid < k) order[tid] = tid;
  __syncthreads();
  if (tid < k && !isfinite(H[tid * ld + tid])) atomicOr(&bad, 1);
  __syncthreads();
  if (tid < k && !bad) {
    const double d = H[tid * ld + tid];
    int rank = 0;
    for (int j = 0; j < k; ++j) {
      const double e = H[j * ld + j];
      rank += (e > d) || (e == d && j < tid);
    }
    order[rank] = tid;
  }
  __syncthreads();
  // V[r][c] = W[order[c]][r]  (the dummy, if any, sorted last and is dropped)
  for (int c = warp; c < kin; c += nw) {
    const double* wr = W + order[c] * ld;
    for (int r = lane; r < kin; r += 32) Vout[r * kin + c] = wr[r];
  }
  if (tid < kin) theta[tid] = H[order[tid] * ld + order[tid]];
  if (tid == 0 && sweeps_out) *sweeps_out = bad ? -1 : sweep;
}

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

// q = y / ||y||  (single CTA)
__global__ void k_normalize(const double* __restrict__ y, int64_t d, double* __restrict__ q) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) s += y[i] * y[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const double inv = red[0] > 0 ? 1.0 / sqrt(red[0]) : 0.0;
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) q[i] = y[i] * inv;
}
// out = {q^T y, ||y - (q^T y) q||} for unit q  (single CTA)
__global__ void k_rayleigh1(const double* __restrict__ q, const double* __restrict__ y, int64_t d,
                            double* __restrict__ out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) s += q[i] * y[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const double th = red[0];
  __syncthreads();
  s = 0.0;
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) {
    const double r = y[i] - th * q[i];
    s += r * r;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = th;
    out[1] = sqrt(red[0]);
  }
}

__global__ void k_count_nonfinite(const double* x, int64_t n, int* out) {
  int c = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    c += !isfinite(x[e]);
  if (c) atomicAdd(out, c);
}

// resid[i] = || SQ[:, i] - theta_i Q[:, i] ||_2, one CTA per column i < ncol
__global__ void k_resid(const double* __restrict__ SQ, const double* __restrict__ Q, int64_t d,
                        int k, const double* __restrict__ theta, double* __restrict__ resid) {
  __shared__ double red[256];
  const int i = blockIdx.x;
  const double t = theta[i];
  double s = 0.0;
  for (int64_t r = threadIdx.x; r < d; r += blockDim.x) {
    const double v = SQ[r * k + i] - t * Q[r * k + i];
    s += v * v;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) resid[i] = sqrt(red[0]);
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// deterministic pseudo-random fill of columns [c0, k) of Q (d x k): uniform(-1, 1)
__global__ void k_fill_random(double* Q, int64_t d, int k, int c0, uint64_t seed) {
  const int64_t n = d * (k - c0);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / (k - c0);
    const int c = c0 + (int)(e % (k - c0));
    const uint64_t h = mix64(seed ^ mix64((uint64_t)r * 1315423911ull + (uint64_t)c));
    Q[r * k + c] = ((double)(h >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
  }
}

// z = alpha x + beta y (z may alias x or y)
__global__ void k_axpby(int64_t n, double alpha, const double* x, double beta, const double* y,
                        double* z) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    z[e] = alpha * x[e] + (beta != 0.0 ? beta * y[e] : 0.0);
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

int choose_block(int J, int64_t d, int oversample) {
  int p = oversample > 0 ? oversample : std::max(8, std::min(J, 32));
  int k = J + p;
  if (k > kMaxBlock) k = kMaxBlock;
  if (k > d) k = (int)d;
  if (k & 1) k = (k + 1 <= kMaxBlock && k + 1 <= d) ? k + 1 : k - 1;
  if (k < J) k = J;
  return k;
}

// Q (d x k) <- Q R^{-1} twice (CholQR2)
void cholqr2_impl(double* Q, int64_t d, int k, EigWs& ws, cudaStream_t st) {
  const size_t smem = (size_t)2 * k * (k + 1) * sizeof(double);
  for (int pass = 0; pass < 2; ++pass) {
    dgemm(k, k, d, 1.0, f64(Q, k, true), f64(Q, k), 0.0, ws.H.p, k, 0.0, nullptr, 0, ws.dense, st);
    launch_chol_inv(ws.H.p, k, ws.R.p, 0.0, st);
    dgemm(d, k, k, 1.0, f64(Q, k), f64(ws.R.p, k), 0.0, ws.T.p, k, 0.0, nullptr, 0, ws.dense, st);
    TK_LAUNCH(k_copy_cols, grid_for(d * k), 256, 0, st, ws.T.p, (int64_t)k, Q, (int64_t)k, d, k);
  }
}

}  // namespace

void cholqr2(double* V, int64_t ldv, int64_t d, int J, EigWs& ws, cudaStream_t st) {
  ws.Q.ensure((size_t)(d * J));
  ws.T.ensure((size_t)(d * J));
  ws.H.ensure((size_t)J * J);
  ws.R.ensure((size_t)J * J);
  TK_LAUNCH(k_copy_cols, grid_for(d * J), 256, 0, st, V, ldv, ws.Q.p, (int64_t)J, d, J);
  cholqr2_impl(ws.Q.p, d, J, ws, st);
  TK_LAUNCH(k_copy_cols, grid_for(d * J), 256, 0, st, ws.Q.p, (int64_t)J, V, ldv, d, J);
}

void canon_to_f32(const double* V, int64_t ldv, int64_t d, int J, float* U, cudaStream_t st) {
  TK_LAUNCH(k_canon_f32, J, 256, 0, st, V, ldv, d, J, U);
}

bool eig_leading(double* S, int64_t lds, int64_t d, int J, EigSlot& slot, EigWs& ws,
                 const EigOpts& o, double* out_V, int64_t ldv, double* theta_out,
                 cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    TK_CUDA(cudaFuncSetAttribute(k_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 2 * kMaxBlock * (kMaxBlock + 1) * (int)sizeof(double)));
    TK_CUDA(cudaFuncSetAttribute(k_chol_inv<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 2 * kMaxBlock * (kMaxBlock + 1) * (int)sizeof(double)));
    TK_CUDA(cudaFuncSetAttribute(k_chol_inv<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 2 * kMaxBlock * (kMaxBlock + 1) * (int)sizeof(double)));
    TK_CUDA(cudaFuncSetAttribute(k_chol_inv<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 2 * kMaxBlock * (kMaxBlock + 1) * (int)sizeof(double)));
    TK_CUDA(cudaFuncSetAttribute(k_chol_inv<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 2 * kMaxBlock * (kMaxBlock + 1) * (int)sizeof(double)));
    attr_set = true;
  }
  if (lds != d) fail(TUCKER_E_ARG, "eig_leading: lds must equal d");
  const int k = choose_block(J, d, o.oversample);
  const size_t dk = (size_t)(d * k);
  // A: active block (d x ka, contiguous, ld = ka) in ws.Q; L: locked vectors (d x J, ld = J)
  ws.Q.ensure(dk);
  ws.SQ.ensure(dk);
  ws.X.ensure(dk);
  ws.Y.ensure(dk);
  ws.T.ensure(dk);
  ws.H.ensure((size_t)k * k);
  ws.V.ensure((size_t)k * k);
  ws.R.ensure((size_t)k * k);
  ws.theta.ensure(k);
  ws.resid.ensure(k);
  ws.L.ensure((size_t)(d * J));
  ws.LT.ensure((size_t)(d * J));
  ws.Z.ensure((size_t)J * k);
  ws.h_theta.assign(k, 0.0);
  ws.h_resid.assign(k, 0.0);
  ws.dsweeps.ensure(1);
  std::vector<double> th_lock;  // Ritz values of the locked vectors
  static const bool dbg = std::getenv("TUCKER_EIG_DEBUG") != nullptr;

  int nlock = 0;
  int ka = k;
  if (slot.valid && slot.d == d && slot.k == k) {
    TK_CUDA(cudaMemcpyAsync(ws.Q.p, slot.basis.p, dk * sizeof(double), cudaMemcpyDeviceToDevice, st));
  } else {
    TK_LAUNCH(k_fill_random, grid_for(d * k), 256, 0, st, ws.Q.p, d, k, 0,
              (uint64_t)0x5eed0000ull + (uint64_t)d * 131 + (uint64_t)J);
  }

  auto nonfinite = [&](const double* x, int64_t n, const char* what) {
    if (!dbg) return;
    TK_CUDA(cudaMemsetAsync(ws.dsweeps.p, 0, sizeof(int), st));
    TK_LAUNCH(k_count_nonfinite, grid_for(n), 256, 0, st, x, n, ws.dsweeps.p);
    int h = 0;
    TK_CUDA(cudaMemcpyAsync(&h, ws.dsweeps.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaStreamSynchronize(st));
    std::fprintf(stderr, "[eig] nonfinite %s: %d of %lld\n", what, h, (long long)n);
  };
  // orthonormalise A (d x ka) against L (d x nlock) and itself (CholQR2, equilibrated)
  auto orth_active = [&](int passes, bool project) {
    if (nlock > 0 && project) {
      for (int pass = 0; pass < 2; ++pass) {
        dgemm(nlock, ka, d, 1.0, f64(ws.L.p, J, true), f64(ws.Q.p, ka), 0.0, ws.Z.p, ka, 0.0,
              nullptr, 0, ws.dense, st);
        dgemm(d, ka, nlock, -1.0, f64(ws.L.p, J), f64(ws.Z.p, ka), 1.0, ws.Q.p, ka, 0.0, nullptr, 0,
              ws.dense, st);
      }
    }
    const size_t smem = (size_t)2 * ka * (ka + 1) * sizeof(double);
    // shifted CholQR3 (first pass shifted so the factorisation cannot break down)
    const double shift = 11.0 * ((double)d * ka + (double)ka * (ka + 1)) * 1.1e-16 * ka;
    for (int pass = 0; pass < passes; ++pass) {
      dgemm(ka, ka, d, 1.0, f64(ws.Q.p, ka, true), f64(ws.Q.p, ka), 0.0, ws.H.p, ka, 0.0, nullptr,
            0, ws.dense, st);
      nonfinite(ws.H.p, (int64_t)ka * ka, "gram-in-orth");
      launch_chol_inv(ws.H.p, ka, ws.R.p, pass == 0 ? shift : 0.0, st);
      nonfinite(ws.R.p, (int64_t)ka * ka, "Rinv");
      dgemm(d, ka, ka, 1.0, f64(ws.Q.p, ka), f64(ws.R.p, ka), 0.0, ws.T.p, ka, 0.0, nullptr, 0,
            ws.dense, st);
      std::swap(ws.Q, ws.T);
    }
  };
  // out = alpha S Y + gamma Dm + delta Em; S is deflated in place when vectors lock
  auto apply_op = [&](const double* Yp, double alpha, double* out, double gamma, const double* Dm,
                      double delta = 0.0, const double* Em = nullptr) {
    dgemm4(d, ka, d, alpha, f64(S, lds), f64(Yp, ka), 0.0, out, ka, gamma, Dm, ka, delta, Em, ka,
           ws.dense, st);
    ++ws.stat_matvec;
  };
  int n_rr = 0;  // Rayleigh-Ritz steps so far (the first one starts from a non-diagonal H)
  auto rayleigh_ritz = [&]() {
    nonfinite(S, d * d, "S");
    nonfinite(ws.Q.p, d * ka, "Q");
    apply_op(ws.Q.p, 1.0, ws.SQ.p, 0.0, nullptr);
    nonfinite(ws.SQ.p, d * ka, "SQ");
    dgemm(ka, ka, d, 1.0, f64(ws.Q.p, ka, true), f64(ws.SQ.p, ka), 0.0, ws.H.p, ka, 0.0, nullptr,
          0, ws.dense, st);
    nonfinite(ws.H.p, (int64_t)ka * ka, "H");
    const int kp = ka + (ka & 1);
    TK_LAUNCH(k_jacobi, 1, 1024, (size_t)2 * kp * (kp + 1) * sizeof(double), st, ws.H.p, ka,
              ws.V.p, ws.theta.p, k == d ? 60 : (n_rr == 0 ? o.jacobi_sweeps + 1 : o.jacobi_sweeps),
              k == d ? 1e-15 : 1e-13, ws.dsweeps.p);
    ++n_rr;
    dgemm(d, ka, ka, 1.0, f64(ws.Q.p, ka), f64(ws.V.p, ka), 0.0, ws.T.p, ka, 0.0, nullptr, 0,
          ws.dense, st);
    std::swap(ws.Q, ws.T);
    dgemm(d, ka, ka, 1.0, f64(ws.SQ.p, ka), f64(ws.V.p, ka), 0.0, ws.T.p, ka, 0.0, nullptr, 0,
          ws.dense, st);
    std::swap(ws.SQ, ws.T);
    TK_LAUNCH(k_resid, ka, 256, 0, st, ws.SQ.p, ws.Q.p, d, ka, ws.theta.p, ws.resid.p);
    int hs = 0;
    TK_CUDA(cudaMemcpyAsync(ws.h_theta.data() + nlock, ws.theta.p, ka * sizeof(double),
                            cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaMemcpyAsync(ws.h_resid.data() + nlock, ws.resid.p, ka * sizeof(double),
                            cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaMemcpyAsync(&hs, ws.dsweeps.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaStreamSynchronize(st));
    if (hs < 0) fail(TUCKER_E_CUDA, "eigensolver breakdown (non-finite Rayleigh quotient)");
    ws.stat_sweeps += hs;
  };
  auto theta1 = [&]() {
    const double t = nlock > 0 ? th_lock[0] : ws.h_theta[0];
    return t > 0 ? t : 1.0;
  };
  // deflate S by the locked columns [n0, n0 + nl) of L (LT holds S L):
  // S <- (I - Ln Ln^T) S (I - Ln Ln^T) = S - Ln W^T - W Ln^T, W = P - Ln (Ln^T P) / 2, P = S Ln
  auto deflate = [&](int n0, int nl) {
    const double* Ln = ws.L.p + n0;
    double* W = ws.X.p;  // d x nl
    TK_LAUNCH(k_copy_cols, grid_for(d * nl), 256, 0, st, ws.LT.p + n0, (int64_t)J, W, (int64_t)nl, d,
              nl);
    dgemm(nl, nl, d, 1.0, f64(Ln, J, true), f64(W, nl), 0.0, ws.Z.p, nl, 0.0, nullptr, 0, ws.dense, st);
    dgemm(d, nl, nl, -0.5, f64(Ln, J), f64(ws.Z.p, nl), 1.0, W, nl, 0.0, nullptr, 0, ws.dense, st);
    dgemm(d, d, nl, -1.0, f64(Ln, J), f64(W, nl, true), 1.0, S, lds, 0.0, nullptr, 0, ws.dense, st);
    dgemm(d, d, nl, -1.0, f64(W, nl), f64(Ln, J, true), 1.0, S, lds, 0.0, nullptr, 0, ws.dense, st);
  };
  // move the converged leading active vectors into L (prefix, descending order)
  auto lock = [&]() {
    int nl = 0;
    const double th1 = theta1();
    while (nlock + nl < J && nl < ka && ws.h_resid[nlock + nl] <= o.tol * th1) ++nl;
    if (nl == 0) return;
    TK_LAUNCH(k_copy_cols, grid_for(d * nl), 256, 0, st, ws.Q.p, (int64_t)ka, ws.L.p + nlock,
              (int64_t)J, d, nl);
    TK_LAUNCH(k_copy_cols, grid_for(d * nl), 256, 0, st, ws.SQ.p, (int64_t)ka, ws.LT.p + nlock,
              (int64_t)J, d, nl);
    for (int i = 0; i < nl; ++i) th_lock.push_back(ws.h_theta[nlock + i]);
    deflate(nlock, nl);
    const int kn = ka - nl;
    if (kn > 0) {
      TK_LAUNCH(k_copy_cols, grid_for(d * kn), 256, 0, st, ws.Q.p + nl, (int64_t)ka, ws.T.p,
                (int64_t)kn, d, kn);
      std::swap(ws.Q, ws.T);
      TK_LAUNCH(k_copy_cols, grid_for(d * kn), 256, 0, st, ws.SQ.p + nl, (int64_t)ka, ws.T.p,
                (int64_t)kn, d, kn);
      std::swap(ws.SQ, ws.T);
    }
    nlock += nl;
    ka = kn;
  };

  // An outlier top eigenvalue (the "mean" direction of these nonnegative tensors,
  // theta_1 / theta_J ~ 10-80) would cap the Chebyshev degree (m_amp) at 1-3: refine
  // its Ritz vector by power iteration (rate theta_2/theta_1) and deflate it first.
  auto power_lock_top = [&]() {
    if (nlock > 0 || ka < 3 || J < 2) return;
    const double t0 = ws.h_theta[0], t1 = ws.h_theta[1];
    if (!(t1 > 0) || t0 < 3.0 * t1) return;
    const double res = ws.h_resid[0] / t0;
    int npow = (int)std::ceil(std::log(std::max(res / o.tol, 1.0)) / -std::log(t1 / t0)) + 1;
    npow = std::min(npow, 40);
    ws.pq.ensure((size_t)d);
    ws.py.ensure((size_t)d);
    ws.pout.ensure(2);
    TK_LAUNCH(k_copy_cols, grid_for(d), 256, 0, st, ws.Q.p, (int64_t)ka, ws.pq.p, (int64_t)1, d, 1);
    for (int i = 0; i < npow; ++i) {
      dgemm(d, 1, d, 1.0, f64(S, lds), f64(ws.pq.p, 1), 0.0, ws.py.p, 1, 0.0, nullptr, 0, ws.dense, st);
      ++ws.stat_matvec;
      TK_LAUNCH(k_normalize, 1, 256, 0, st, ws.py.p, d, ws.pq.p);
    }
    dgemm(d, 1, d, 1.0, f64(S, lds), f64(ws.pq.p, 1), 0.0, ws.py.p, 1, 0.0, nullptr, 0, ws.dense, st);
    TK_LAUNCH(k_rayleigh1, 1, 256, 0, st, ws.pq.p, ws.py.p, d, ws.pout.p);
    double ho[2];
    TK_CUDA(cudaMemcpyAsync(ho, ws.pout.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaStreamSynchronize(st));
    if (!(ho[1] <= o.tol * ho[0])) return;
    TK_LAUNCH(k_copy_cols, grid_for(d), 256, 0, st, ws.pq.p, (int64_t)1, ws.L.p, (int64_t)J, d, 1);
    TK_LAUNCH(k_copy_cols, grid_for(d), 256, 0, st, ws.py.p, (int64_t)1, ws.LT.p, (int64_t)J, d, 1);
    th_lock.push_back(ho[0]);
    ws.h_theta[0] = ho[0];
    ws.h_resid[0] = ho[1];
    deflate(0, 1);
    // the rest of the block (columns 1..ka-1) becomes the active block
    const int kn = ka - 1;
    TK_LAUNCH(k_copy_cols, grid_for(d * kn), 256, 0, st, ws.Q.p + 1, (int64_t)ka, ws.T.p, (int64_t)kn,
              d, kn);
    std::swap(ws.Q, ws.T);
    nlock = 1;
    ka = kn;
    orth_active(2, true);
    rayleigh_ritz();
    lock();
  };

  orth_active(2, true);
  rayleigh_ritz();
  lock();
  power_lock_top();
  bool converged = nlock >= J || k == d;
  for (int outer = 0; outer < o.max_outer && !converged; ++outer) {
    ++ws.stat_outer;
    const double th1 = theta1();
    const double thJ = ws.h_theta[J - 1];
    const double thtop = ws.h_theta[nlock];  // largest active Ritz value
    double b = ws.h_theta[k - 1];
    if (!(b > 0)) b = 1e-12 * th1;
    if (thJ <= b * (1 + 1e-12)) b = thJ * (1 - 1e-3);
    const double a = 0.0;
    const double e = (b - a) / 2, c = (b + a) / 2;
    const double xJ = std::max((thJ - c) / e, 1.0 + 1e-12);
    const double xt = std::max((thtop - c) / e, xJ);
    const double rJ = std::acosh(xJ), rt = std::acosh(xt);
    double rmax = 0;
    for (int i = nlock; i < J; ++i) rmax = std::max(rmax, ws.h_resid[i] / th1);
    // total degree: enough to reach tol (capped), applied in segments of <= m_amp degrees
    // with an orthonormalisation between them so the block stays inside CholQR's reach
    int m_need = (int)std::ceil(std::log(std::max(rmax / o.tol, 4.0)) / std::max(rJ, 1e-6));
    // the block's bottom Ritz directions (x ~ 1) must stay representable next to the top one:
    // T_m(x_top) <= 2e7 keeps the filtered block inside CholQR's reach (kappa^2 <~ 1e15)
    const int m_amp = std::max(1, std::min(16, (int)std::floor(std::log(2e7) / std::max(rt, 1e-6))));
    // few segments when the top direction limits the degree: re-run Rayleigh-Ritz soon so the
    // dominant vectors lock (deflation then lifts m_amp)
    m_need = std::max(1, std::min(std::min(m_need, 64), (m_amp < 6 ? 2 : 8) * m_amp));
    const int m = m_need;
    for (int done = 0; done < m_need;) {
      const int mseg = std::min(m_amp, m_need - done);
      // scaled Chebyshev recurrence (Zhou & Saad) damping [a, b], normalised at thtop
      double sigma = e / (thtop - c);
      const double tau = 2.0 / sigma;
      // Y1 = (S_defl A - c A) sigma / e ; S_defl A = SQ after a Rayleigh-Ritz step
      if (done > 0) apply_op(ws.Q.p, 1.0, ws.SQ.p, 0.0, nullptr);
      TK_LAUNCH(k_axpby, grid_for(d * ka), 256, 0, st, d * ka, sigma / e, ws.SQ.p, -c * sigma / e,
                ws.Q.p, ws.Y.p);
      double* Xp = ws.Q.p;  // T_{i-2}
      double* Yp = ws.Y.p;  // T_{i-1}
      double* spare[2] = {ws.X.p, ws.T.p};
      int si = 0;
      for (int i = 2; i <= mseg; ++i) {
        const double sigma2 = 1.0 / (tau - sigma);
        // T_i = 2 sigma2 / e (S T_{i-1} - c T_{i-1}) - sigma sigma2 T_{i-2}  (one fused GEMM)
        double* Tp = spare[si];
        apply_op(Yp, 2 * sigma2 / e, Tp, -sigma * sigma2, Xp, -2 * sigma2 * c / e, Yp);
        spare[si] = Xp;
        si ^= 1;
        Xp = Yp;
        Yp = Tp;
        sigma = sigma2;
      }
      // the filtered block becomes the active block Q
      if (Yp != ws.Q.p) {
        DBuf<double>* own = (Yp == ws.X.p) ? &ws.X : (Yp == ws.Y.p) ? &ws.Y : &ws.T;
        std::swap(ws.Q, *own);
      }
      done += mseg;
      if (done < m_need) orth_active(1, false);
    }
    orth_active(2, true);
    rayleigh_ritz();
    if (dbg) {
      std::fprintf(stderr, "[eig] d=%lld J=%d k=%d outer=%d m=%d(amp %d) nlock=%d ka=%d rmax=%.3e th1=%.6e thJ=%.6e thtop=%.6e b=%.6e\n",
                   (long long)d, J, k, outer, m, m_amp, nlock, ka, rmax, th1, thJ, thtop, b);
      for (int i = nlock; i < std::min(k, nlock + 4); ++i)
        std::fprintf(stderr, "    th[%d]=%.6e res=%.3e\n", i, ws.h_theta[i], ws.h_resid[i]);
    }
    lock();
    converged = nlock >= J;
  }
  // outputs: the J leading columns of [L | A], sorted by Ritz value (descending)
  std::vector<double> th_all(th_lock);
  for (int i = 0; i < ka; ++i) th_all.push_back(ws.h_theta[nlock + i]);
  std::vector<int> ord(k);
  for (int i = 0; i < k; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return th_all[x] > th_all[y]; });
  for (int j = 0; j < J; ++j) {
    const int src = ord[j];
    if (src < nlock)
      TK_LAUNCH(k_copy_cols, grid_for(d), 256, 0, st, ws.L.p + src, (int64_t)J, out_V + j, ldv, d, 1);
    else
      TK_LAUNCH(k_copy_cols, grid_for(d), 256, 0, st, ws.Q.p + (src - nlock), (int64_t)ka,
                out_V + j, ldv, d, 1);
    theta_out[j] = th_all[src];
  }
  // warm-start basis [L | A] for the next solve of this slot
  slot.basis.ensure(dk);
  if (nlock > 0)
    TK_LAUNCH(k_copy_cols, grid_for(d * nlock), 256, 0, st, ws.L.p, (int64_t)J, slot.basis.p,
              (int64_t)k, d, nlock);
  if (ka > 0)
    TK_LAUNCH(k_copy_cols, grid_for(d * ka), 256, 0, st, ws.Q.p, (int64_t)ka,
              slot.basis.p + nlock, (int64_t)k, d, ka);
  slot.d = d;
  slot.k = k;
  slot.valid = true;
  TK_CUDA(cudaStreamSynchronize(st));
  return converged;
}

}  // namespace tk
