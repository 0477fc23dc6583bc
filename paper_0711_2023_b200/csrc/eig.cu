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
// One CTA.  H (k x k, row-major, ldh) -> V (k x k) eigenvectors in columns and
// theta (k) eigenvalues, sorted descending.  k even, k <= kMaxBlock.
__global__ void __launch_bounds__(1024) k_jacobi(const double* __restrict__ Hin, int k,
                                                 double* __restrict__ Vout,
                                                 double* __restrict__ theta, int max_sweeps,
                                                 int* sweeps_out) {
  extern __shared__ double sm[];
  double* H = sm;          // k*k
  double* V = sm + k * k;  // k*k
  __shared__ double cs_c[kMaxBlock / 2], cs_s[kMaxBlock / 2];
  __shared__ int top[kMaxBlock / 2], bot[kMaxBlock / 2], act[kMaxBlock / 2];
  __shared__ int pos[kMaxBlock], npos[kMaxBlock];
  __shared__ int order[kMaxBlock];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int np = k / 2;
  for (int e = tid; e < k * k; e += nt) {
    const int r = e / k, c = e % k;
    H[e] = 0.5 * (Hin[r * k + c] + Hin[c * k + r]);
    V[e] = (r == c) ? 1.0 : 0.0;
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
        const double app = H[p * k + p], aqq = H[q * k + q], apq = H[p * k + q];
        double c = 1.0, s = 0.0;
        if (apq != 0.0 && fabs(apq) > 1e-15 * sqrt(fabs(app * aqq))) {
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
      if (any) {
        any_in_sweep = 1;
        // two-sided update of every 2x2 block (P <= Q) touched by an active rotation
        for (int b = tid; b < np * np; b += nt) {
          const int P = b / np, Q = b % np;
          if (P > Q || (!act[P] && !act[Q])) continue;
          const int p1 = top[P], p2 = bot[P], q1 = top[Q], q2 = bot[Q];
          const double cP = cs_c[P], sP = cs_s[P], cQ = cs_c[Q], sQ = cs_s[Q];
          if (P == Q) {
            const double app = H[p1 * k + p1], aqq = H[p2 * k + p2], apq = H[p1 * k + p2];
            if (act[P]) {
              const double t = sP / cP;
              H[p1 * k + p1] = app - t * apq;
              H[p2 * k + p2] = aqq + t * apq;
              H[p1 * k + p2] = 0.0;
              H[p2 * k + p1] = 0.0;
            }
            continue;
          }
          double b11 = H[p1 * k + q1], b12 = H[p1 * k + q2];
          double b21 = H[p2 * k + q1], b22 = H[p2 * k + q2];
          // rows: J_P^T
          double r11 = cP * b11 - sP * b21, r12 = cP * b12 - sP * b22;
          double r21 = sP * b11 + cP * b21, r22 = sP * b12 + cP * b22;
          // cols: J_Q
          b11 = r11 * cQ - r12 * sQ;
          b12 = r11 * sQ + r12 * cQ;
          b21 = r21 * cQ - r22 * sQ;
          b22 = r21 * sQ + r22 * cQ;
          H[p1 * k + q1] = b11; H[q1 * k + p1] = b11;
          H[p1 * k + q2] = b12; H[q2 * k + p1] = b12;
          H[p2 * k + q1] = b21; H[q1 * k + p2] = b21;
          H[p2 * k + q2] = b22; H[q2 * k + p2] = b22;
        }
        for (int e = tid; e < np * k; e += nt) {
          const int P = e / k, r = e % k;
          if (!act[P]) continue;
          const int p1 = top[P], p2 = bot[P];
          const double c = cs_c[P], s = cs_s[P];
          const double x = V[r * k + p1], y = V[r * k + p2];
          V[r * k + p1] = x * c - y * s;
          V[r * k + p2] = x * s + y * c;
        }
      }
      __syncthreads();
      // circle-method tournament: keep pos[0], rotate the rest
      if (tid < k) npos[tid] = (tid == 0) ? pos[0] : pos[tid == 1 ? k - 1 : tid - 1];
      __syncthreads();
      if (tid < k) pos[tid] = npos[tid];
      __syncthreads();
    }
    if (!any_in_sweep) break;
  }
  // sort eigenvalues descending (stable by index): rank of each diagonal entry
  __shared__ int bad;
  if (tid == 0) bad = 0;
  if (tid < k) order[tid] = tid;
  __syncthreads();
  if (tid < k && !isfinite(H[tid * k + tid])) atomicOr(&bad, 1);
  __syncthreads();
  if (tid < k && !bad) {
    const double d = H[tid * k + tid];
    int rank = 0;
    for (int j = 0; j < k; ++j) {
      const double e = H[j * k + j];
      rank += (e > d) || (e == d && j < tid);
    }
    order[rank] = tid;
  }
  __syncthreads();
  for (int e = tid; e < k * k; e += nt) {
    const int r = e / k, c = e % k;
    Vout[r * k + c] = V[r * k + order[c]];
  }
  if (tid < k) theta[tid] = H[order[tid] * k + order[tid]];
  if (tid == 0 && sweeps_out) *sweeps_out = bad ? -1 : sweep;
}

// ------------------------------------------------------- Cholesky / inverse --
// One CTA.  G (k x k SPD) -> Rinv (k x k upper triangular) with G = R^T R.
__global__ void __launch_bounds__(1024) k_chol_inv(const double* __restrict__ G, int k,
                                                   double* __restrict__ Rinv, double shift) {
  extern __shared__ double sm[];
  double* A = sm;  // k*k
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ double maxd;
  __shared__ double dsc[kMaxBlock];
  for (int i = tid; i < k; i += nt) {
    const double g = G[i * k + i];
    dsc[i] = g > 0 ? 1.0 / sqrt(g) : 1.0;
  }
  __syncthreads();
  for (int e = tid; e < k * k; e += nt)
    A[e] = G[e] * dsc[e / k] * dsc[e % k] + ((e / k == e % k) ? shift : 0.0);
  __syncthreads();
  if (tid == 0) maxd = 1.0;
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    if (tid == 0) {
      double d = A[j * k + j];
      const double floor = 1e-12 * maxd;
      A[j * k + j] = sqrt(d > floor ? d : floor);
    }
    __syncthreads();
    const double piv = A[j * k + j];
    for (int l = j + 1 + tid; l < k; l += nt) A[j * k + l] /= piv;
    __syncthreads();
    const int w = k - j - 1;
    for (int e = tid; e < w * w; e += nt) {
      const int l = j + 1 + e / w, m = j + 1 + e % w;
      if (m >= l) A[l * k + m] -= A[j * k + l] * A[j * k + m];
    }
    __syncthreads();
  }
  // R = upper(A).  Solve R X = I column by column (thread c owns column c).
  for (int c = tid; c < k; c += nt) {
    for (int i = k - 1; i >= 0; --i) {
      double x;
      if (i > c) {
        x = 0.0;
      } else {
        double s = (i == c) ? 1.0 : 0.0;
        for (int l = i + 1; l <= c; ++l) s -= A[i * k + l] * Rinv[l * k + c];
        x = s / A[i * k + i];
      }
      Rinv[i * k + c] = x;
    }
  }
  __syncthreads();
  for (int e = tid; e < k * k; e += nt) Rinv[e] *= dsc[e / k];
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
  const size_t smem = (size_t)k * k * sizeof(double);
  for (int pass = 0; pass < 2; ++pass) {
    dgemm(k, k, d, 1.0, f64(Q, k, true), f64(Q, k), 0.0, ws.H.p, k, 0.0, nullptr, 0, ws.dense, st);
    TK_LAUNCH(k_chol_inv, 1, 512, smem, st, ws.H.p, k, ws.R.p, 0.0);
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
                                 2 * kMaxBlock * kMaxBlock * (int)sizeof(double)));
    TK_CUDA(cudaFuncSetAttribute(k_chol_inv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kMaxBlock * kMaxBlock * (int)sizeof(double) + 1024));
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
    const size_t smem = (size_t)ka * ka * sizeof(double);
    // shifted CholQR3 (first pass shifted so the factorisation cannot break down)
    const double shift = 11.0 * ((double)d * ka + (double)ka * (ka + 1)) * 1.1e-16 * ka;
    for (int pass = 0; pass < 3; ++pass) {
      dgemm(ka, ka, d, 1.0, f64(ws.Q.p, ka, true), f64(ws.Q.p, ka), 0.0, ws.H.p, ka, 0.0, nullptr,
            0, ws.dense, st);
      nonfinite(ws.H.p, (int64_t)ka * ka, "gram-in-orth");
      TK_LAUNCH(k_chol_inv, 1, 512, smem, st, ws.H.p, ka, ws.R.p, pass == 0 ? shift : 0.0);
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
    TK_LAUNCH(k_jacobi, 1, 1024, (size_t)2 * ka * ka * sizeof(double), st, ws.H.p, ka, ws.V.p,
              ws.theta.p, 40, ws.dsweeps.p);
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
