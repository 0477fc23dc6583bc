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
// Parallel cyclic Jacobi (circle-method tournament: k/2 disjoint rotations per
// round, k-1 rounds per sweep).  H and V live in shared memory with an odd row
// stride (k+1) against bank conflicts.  Rotations with
// |h_pq| <= tol * sqrt(h_pp h_qq) are skipped; the sweep loop stops when a sweep
// makes no rotation or after max_sweeps (the caller's Ritz residuals decide
// convergence, so a capped solve only costs another outer iteration).
__global__ void __launch_bounds__(1024) k_jacobi(const double* __restrict__ Hin, int k,
                                                 double* __restrict__ Vout,
                                                 double* __restrict__ theta, int max_sweeps,
                                                 double tol, int* sweeps_out) {
  extern __shared__ double sm[];
  const int ld = k + 1;
  double* H = sm;           // k x ld
  double* V = sm + k * ld;  // k x ld
  __shared__ double cs_c[kMaxBlock / 2], cs_s[kMaxBlock / 2];
  __shared__ int top[kMaxBlock / 2], bot[kMaxBlock / 2], act[kMaxBlock / 2];
  __shared__ int pos[kMaxBlock];
  __shared__ int order[kMaxBlock];
  __shared__ int bad;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int np = k / 2;
  for (int r = warp; r < k; r += 32)
    for (int c = lane; c < k; c += 32) {
      H[r * ld + c] = 0.5 * (Hin[r * k + c] + Hin[c * k + r]);
      V[r * ld + c] = (r == c) ? 1.0 : 0.0;
    }
  for (int i = tid; i < k; i += nt) pos[i] = i;
  __syncthreads();
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    int any_in_sweep = 0;
    for (int round = 0; round < k - 1; ++round) {
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
        // two-sided update of the 2x2 blocks (P <= Q): warp -> P, lane -> Q
        for (int P = warp; P < np; P += 32) {
          const int p1 = top[P], p2 = bot[P];
          const double cP = cs_c[P], sP = cs_s[P];
          const int aP = act[P];
          for (int Q = lane; Q < np; Q += 32) {
            if (Q < P || (!aP && !act[Q])) continue;
            if (Q == P) {
              if (aP) {
                const double apq = H[p1 * ld + p2];
                const double t = sP / cP;
                H[p1 * ld + p1] -= t * apq;
                H[p2 * ld + p2] += t * apq;
                H[p1 * ld + p2] = 0.0;
                H[p2 * ld + p1] = 0.0;
              }
              continue;
            }
            const int q1 = top[Q], q2 = bot[Q];
            const double cQ = cs_c[Q], sQ = cs_s[Q];
            const double b11 = H[p1 * ld + q1], b12 = H[p1 * ld + q2];
            const double b21 = H[p2 * ld + q1], b22 = H[p2 * ld + q2];
            const double r11 = cP * b11 - sP * b21, r12 = cP * b12 - sP * b22;
            const double r21 = sP * b11 + cP * b21, r22 = sP * b12 + cP * b22;
            const double n11 = r11 * cQ - r12 * sQ, n12 = r11 * sQ + r12 * cQ;
            const double n21 = r21 * cQ - r22 * sQ, n22 = r21 * sQ + r22 * cQ;
            H[p1 * ld + q1] = n11; H[q1 * ld + p1] = n11;
            H[p1 * ld + q2] = n12; H[q2 * ld + p1] = n12;
            H[p2 * ld + q1] = n21; H[q1 * ld + p2] = n21;
            H[p2 * ld + q2] = n22; H[q2 * ld + p2] = n22;
          }
        }
        // V <- V J: warp -> pair P, lane -> rows
        for (int P = warp; P < np; P += 32) {
          if (!act[P]) continue;
          const int p1 = top[P], p2 = bot[P];
          const double c = cs_c[P], s = cs_s[P];
          for (int r = lane; r < k; r += 32) {
            const double x = V[r * ld + p1], y = V[r * ld + p2];
            V[r * ld + p1] = x * c - y * s;
            V[r * ld + p2] = x * s + y * c;
          }
        }
      }
      __syncthreads();
      if (tid < k) pos[tid] = nextpos;  // circle-method tournament: keep pos[0], rotate the rest
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
  for (int r = warp; r < k; r += 32)
    for (int c = lane; c < k; c += 32) Vout[r * k + c] = V[r * ld + order[c]];
  if (tid < k) theta[tid] = H[order[tid] * ld + order[tid]];
  if (tid == 0 && sweeps_out) *sweeps_out = bad ? -1 : sweep;
}

// ------------------------------------------------------- Cholesky / inverse --
// One CTA of 256 threads.  G (k x k SPD, equilibrated to unit diagonal first,
// plus `shift` on the diagonal) -> Rinv (k x k upper) with D G D + shift I = R^T R
// and Rinv = D R^{-1}, so Y Rinv has orthonormal columns when G = Y^T Y.
__global__ void __launch_bounds__(256) k_chol_inv(const double* __restrict__ G, int k,
                                                   double* __restrict__ Rinv, double shift) {
  extern __shared__ double sm[];
  const int ld = k + 1;
  double* A = sm;           // k x ld : R (upper)
  double* X = sm + k * ld;  // k x ld : R^{-1}
  __shared__ double dsc[kMaxBlock];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < k; i += nt) {
    const double g = G[i * k + i];
    dsc[i] = g > 0 ? 1.0 / sqrt(g) : 1.0;
  }
  __syncthreads();
  for (int r = warp; r < k; r += (nt >> 5))
    for (int c = lane; c < k; c += 32) {
      A[r * ld + c] = G[r * k + c] * dsc[r] * dsc[c] + (r == c ? shift : 0.0);
      X[r * ld + c] = 0.0;
    }
  __syncthreads();
  // right-looking Cholesky, upper triangle: row j of R = row j / sqrt(pivot)
  for (int j = 0; j < k; ++j) {
    const double dj = A[j * ld + j];
    const double piv = sqrt(dj > 1e-12 ? dj : 1e-12);
    __syncthreads();
    for (int l = j + tid; l < k; l += nt) A[j * ld + l] = (l == j) ? piv : A[j * ld + l] / piv;
    __syncthreads();
    const int w = k - j - 1;
    // trailing update of the upper triangle: warp -> rows, lane -> cols
    for (int l = j + 1 + warp; l < k; l += (nt >> 5)) {
      const double ajl = A[j * ld + l];
      for (int m = l + lane; m < k; m += 32) A[l * ld + m] -= ajl * A[j * ld + m];
    }
    (void)w;
    __syncthreads();
  }
  // X = R^{-1}, rows from the bottom: X[i][j] = -(1/R_ii) sum_{l=i+1..j} R[i][l] X[l][j].
  // 2 threads per column j (k <= 116 <= 128 columns), shuffle-reduced.
  for (int i = k - 1; i >= 0; --i) {
    const double rii = A[i * ld + i];
    const int j = i + (tid >> 1);
    const int sub = tid & 1;
    double s = 0.0;
    if (j < k && j > i)
      for (int l = i + 1 + sub; l <= j; l += 2) s += A[i * ld + l] * X[l * ld + j];
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (sub == 0 && j < k) X[i * ld + j] = (j == i) ? 1.0 / rii : -s / rii;
    __syncthreads();
  }
  for (int r = warp; r < k; r += (nt >> 5))
    for (int c = lane; c < k; c += 32) Rinv[r * k + c] = dsc[r] * X[r * ld + c];
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
    TK_LAUNCH(k_chol_inv, 1, 256, smem, st, ws.H.p, k, ws.R.p, 0.0);
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

bool eig_leading(const double* S, int64_t lds, int64_t d, int J, EigSlot& slot, EigWs& ws,
                 const EigOpts& o, double* out_V, int64_t ldv, double* theta_out,
                 cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    TK_CUDA(cudaFuncSetAttribute(k_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 2 * kMaxBlock * (kMaxBlock + 1) * (int)sizeof(double)));
    TK_CUDA(cudaFuncSetAttribute(k_chol_inv, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
  auto orth_active = [&]() {
    if (nlock > 0) {
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
    for (int pass = 0; pass < 3; ++pass) {
      dgemm(ka, ka, d, 1.0, f64(ws.Q.p, ka, true), f64(ws.Q.p, ka), 0.0, ws.H.p, ka, 0.0, nullptr,
            0, ws.dense, st);
      nonfinite(ws.H.p, (int64_t)ka * ka, "gram-in-orth");
      TK_LAUNCH(k_chol_inv, 1, 256, smem, st, ws.H.p, ka, ws.R.p, pass == 0 ? shift : 0.0);
      nonfinite(ws.R.p, (int64_t)ka * ka, "Rinv");
      dgemm(d, ka, ka, 1.0, f64(ws.Q.p, ka), f64(ws.R.p, ka), 0.0, ws.T.p, ka, 0.0, nullptr, 0,
            ws.dense, st);
      std::swap(ws.Q, ws.T);
    }
  };
  // out = alpha S_defl Y + gamma Dm, S_defl = S - L Theta_L L^T (LT holds S L = L Theta_L + R_L)
  auto apply_op = [&](const double* Yp, double alpha, double* out, double gamma, const double* Dm) {
    dgemm(d, ka, d, alpha, f64(S, lds), f64(Yp, ka), 0.0, out, ka, gamma, Dm, ka, ws.dense, st);
    ++ws.stat_matvec;
    if (nlock > 0) {
      dgemm(nlock, ka, d, 1.0, f64(ws.LT.p, J, true), f64(Yp, ka), 0.0, ws.Z.p, ka, 0.0, nullptr,
            0, ws.dense, st);
      dgemm(d, ka, nlock, -alpha, f64(ws.L.p, J), f64(ws.Z.p, ka), 1.0, out, ka, 0.0, nullptr, 0,
            ws.dense, st);
    }
  };
  auto rayleigh_ritz = [&]() {
    nonfinite(S, d * d, "S");
    nonfinite(ws.Q.p, d * ka, "Q");
    apply_op(ws.Q.p, 1.0, ws.SQ.p, 0.0, nullptr);
    nonfinite(ws.SQ.p, d * ka, "SQ");
    dgemm(ka, ka, d, 1.0, f64(ws.Q.p, ka, true), f64(ws.SQ.p, ka), 0.0, ws.H.p, ka, 0.0, nullptr,
          0, ws.dense, st);
    nonfinite(ws.H.p, (int64_t)ka * ka, "H");
    TK_LAUNCH(k_jacobi, 1, 1024, (size_t)2 * ka * (ka + 1) * sizeof(double), st, ws.H.p, ka,
              ws.V.p, ws.theta.p, k == d ? 60 : o.jacobi_sweeps, k == d ? 1e-15 : 1e-13,
              ws.dsweeps.p);
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
  // move the converged leading active vectors into L (prefix, descending order)
  auto lock = [&]() {
    int nl = 0;
    const double th1 = theta1();
    while (nlock + nl < J && nl < ka && ws.h_resid[nlock + nl] <= o.tol * th1) ++nl;
    if (nlock + nl < J) nl &= ~1;  // keep the active block even (Jacobi pairs all indices)
    if (nl == 0) return;
    TK_LAUNCH(k_copy_cols, grid_for(d * nl), 256, 0, st, ws.Q.p, (int64_t)ka, ws.L.p + nlock,
              (int64_t)J, d, nl);
    TK_LAUNCH(k_copy_cols, grid_for(d * nl), 256, 0, st, ws.SQ.p, (int64_t)ka, ws.LT.p + nlock,
              (int64_t)J, d, nl);
    for (int i = 0; i < nl; ++i) th_lock.push_back(ws.h_theta[nlock + i]);
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

  orth_active();
  rayleigh_ritz();
  lock();
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
    // degree: enough to reach tol, while the top active direction outgrows the J-th by <= 1e8
    int m = (int)std::ceil(std::log(std::max(rmax / o.tol, 4.0)) / std::max(rJ, 1e-6));
    // the block's bottom Ritz directions (x ~ 1) must stay representable next to the top one:
    // T_m(x_top) <= 1e7 keeps the filtered block inside CholQR's reach (kappa^2 <~ 1e14)
    const int m_amp = (int)std::floor(std::log(2e7) / std::max(rt, 1e-6));
    m = std::max(1, std::min(std::min(m, m_amp), 16));
    // scaled Chebyshev recurrence (Zhou & Saad) damping [a, b], normalised at thtop
    double sigma = e / (thtop - c);
    const double tau = 2.0 / sigma;
    // Y1 = (S_defl A - c A) sigma / e, where S_defl A = SQ (A is orthogonal to L)
    TK_LAUNCH(k_axpby, grid_for(d * ka), 256, 0, st, d * ka, sigma / e, ws.SQ.p, -c * sigma / e,
              ws.Q.p, ws.Y.p);
    TK_LAUNCH(k_axpby, grid_for(d * ka), 256, 0, st, d * ka, 1.0, ws.Q.p, 0.0, ws.Q.p, ws.X.p);
    for (int i = 2; i <= m; ++i) {
      const double sigma2 = 1.0 / (tau - sigma);
      // T = 2 sigma2 / e (S_defl Y - c Y) - sigma sigma2 X
      apply_op(ws.Y.p, 2 * sigma2 / e, ws.T.p, -sigma * sigma2, ws.X.p);
      TK_LAUNCH(k_axpby, grid_for(d * ka), 256, 0, st, d * ka, 1.0, ws.T.p, -2 * sigma2 * c / e,
                ws.Y.p, ws.T.p);
      std::swap(ws.X, ws.Y);
      std::swap(ws.Y, ws.T);
      sigma = sigma2;
    }
    std::swap(ws.Q, ws.Y);
    orth_active();
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
