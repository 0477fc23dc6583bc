// dense.cu -- small fp64 dense kernels (eigensolver filter products, CholQR,
// Rayleigh-Ritz projections, core G_(N) = U_N^T Y_(N)).
//
// C = alpha * op(A) op(B) + beta * C + gamma * D, fp64 accumulation, with
// operands stored as fp64, fp32 or split fp32 (hi + lo).  Split-K partials are
// reduced in a fixed order (deterministic).
#include "internal.cuh"

namespace tk {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;

template <Elt E>
struct Ld;
template <>
struct Ld<Elt::F64> {
  __device__ __forceinline__ static double at(const MatRef& r, int64_t off) {
    return __ldg((const double*)r.p + off);
  }
};
template <>
struct Ld<Elt::F32> {
  __device__ __forceinline__ static double at(const MatRef& r, int64_t off) {
    return (double)__ldg((const float*)r.p + off);
  }
};
template <>
struct Ld<Elt::SPLIT> {
  __device__ __forceinline__ static double at(const MatRef& r, int64_t off) {
    return (double)__ldg((const float*)r.p + off) + (double)__ldg(r.lo + off);
  }
};

struct GemmArgs {
  int64_t M, N, K;
  MatRef A, B;
  double alpha, beta, gamma;
  double* C;
  int64_t ldc;
  const double* D;
  int64_t ldd;
  double delta;
  const double* E;
  int64_t lde;
  double* part;  // split-K partials [splits][M][N] or null
  int64_t kchunk;
};

template <Elt EA, Elt EB>
__global__ void __launch_bounds__(256) k_dgemm(GemmArgs g) {
  __shared__ double As[BK][BM + 1];
  __shared__ double Bs[BK][BN + 1];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int64_t kb = (int64_t)blockIdx.z * g.kchunk;
  const int64_t ke = min(g.K, kb + g.kchunk);
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int64_t k0 = kb; k0 < ke; k0 += BK) {
    // A tile: op(A)[m][k]
#pragma unroll
    for (int t = 0; t < (BM * BK) / 256; ++t) {
      const int e = tid + 256 * t;
      int mm, kk;
      if (g.A.trans) { mm = e % BM; kk = e / BM; } else { kk = e % BK; mm = e / BK; }
      const int64_t m = m0 + mm, k = k0 + kk;
      double v = 0.0;
      if (m < g.M && k < ke) v = Ld<EA>::at(g.A, g.A.trans ? k * g.A.ld + m : m * g.A.ld + k);
      As[kk][mm] = v;
    }
#pragma unroll
    for (int t = 0; t < (BN * BK) / 256; ++t) {
      const int e = tid + 256 * t;
      int nn, kk;
      if (g.B.trans) { kk = e % BK; nn = e / BK; } else { nn = e % BN; kk = e / BN; }
      const int64_t n = n0 + nn, k = k0 + kk;
      double v = 0.0;
      if (n < g.N && k < ke) v = Ld<EB>::at(g.B, g.B.trans ? n * g.B.ld + k : k * g.B.ld + n);
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
      if (m >= g.M || n >= g.N) continue;
      if (g.part) {
        g.part[((int64_t)blockIdx.z * g.M + m) * g.N + n] = acc[i][j];
      } else {
        double c = g.alpha * acc[i][j];
        if (g.beta != 0.0) c += g.beta * g.C[m * g.ldc + n];
        if (g.gamma != 0.0) c += g.gamma * g.D[m * g.ldd + n];
        if (g.delta != 0.0) c += g.delta * g.E[m * g.lde + n];
        g.C[m * g.ldc + n] = c;
      }
    }
}

__global__ void k_splitk_reduce(int64_t M, int64_t N, int splits, const double* __restrict__ part,
                                double alpha, double beta, double* C, int64_t ldc, double gamma,
                                const double* D, int64_t ldd, double delta, const double* E,
                                int64_t lde) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < M * N;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e / N, n = e % N;
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += part[(int64_t)z * M * N + e];
    double c = alpha * s;
    if (beta != 0.0) c += beta * C[m * ldc + n];
    if (gamma != 0.0) c += gamma * D[m * ldd + n];
    if (delta != 0.0) c += delta * E[m * lde + n];
    C[m * ldc + n] = c;
  }
}


// ---------------------------------------------------------------------------
// NN fast path for the eigensolver's tall products C (M x N) = A (M x K) B (K x N),
// fp64 row-major, N <= 128: CTA tile 64 x BN (BN = 32 * NC), BK = 16, 256 threads,
// 8 rows x NC cols per thread, double-buffered cp.async staging.  Split-K over
// blockIdx.z writes partials (reduced in a fixed order by k_splitk_reduce).
// ---------------------------------------------------------------------------
constexpr int NBM = 64, NBK = 16;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int NC>
__global__ void __launch_bounds__(256) k_dgemm_nn(GemmArgs g) {
  constexpr int BN = 32 * NC;
  __shared__ __align__(16) double As[2][NBK][NBM];
  __shared__ __align__(16) double Bs[2][NBK][BN];
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int64_t m0 = (int64_t)blockIdx.y * NBM;
  const int64_t kb = (int64_t)blockIdx.z * g.kchunk;
  const int64_t ke = min(g.K, kb + g.kchunk);
  const double* A = (const double*)g.A.p;
  const double* B = (const double*)g.B.p;
  auto load = [&](int buf, int64_t k0) {
    // A tile 64 x 16 (row-major along K) -> As[k][m]
#pragma unroll
    for (int t = 0; t < (NBM * NBK) / 256; ++t) {
      const int e = tid + 256 * t;
      const int kk = e % NBK, mm = e / NBK;
      const int64_t m = m0 + mm, k = k0 + kk;
      const bool ok = m < g.M && k < ke;
      cp_async8(&As[buf][kk][mm], ok ? A + m * g.A.ld + k : A, ok);
    }
#pragma unroll
    for (int t = 0; t < (BN * NBK) / 256; ++t) {
      const int e = tid + 256 * t;
      const int nn = e % BN, kk = e / BN;
      const int64_t k = k0 + kk;
      const bool ok = nn < g.N && k < ke;
      cp_async8(&Bs[buf][kk][nn], ok ? B + k * g.B.ld + nn : B, ok);
    }
    cp_async_commit();
  };
  double acc[8][NC];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < NC; ++j) acc[i][j] = 0.0;
  int buf = 0;
  if (kb < ke) load(0, kb);
  for (int64_t k0 = kb; k0 < ke; k0 += NBK) {
    cp_async_wait0();
    __syncthreads();
    if (k0 + NBK < ke) load(buf ^ 1, k0 + NBK);
#pragma unroll
    for (int kk = 0; kk < NBK; ++kk) {
      double a[8], b[NC];
      const double2* ap = reinterpret_cast<const double2*>(&As[buf][kk][ty * 8]);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double2 v = ap[i];
        a[2 * i] = v.x;
        a[2 * i + 1] = v.y;
      }
#pragma unroll
      for (int j = 0; j < NC; ++j) b[j] = Bs[buf][kk][tx + 32 * j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < NC; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const int64_t m = m0 + ty * 8 + i, n = tx + 32 * j;
      if (m >= g.M || n >= g.N) continue;
      if (g.part) {
        g.part[((int64_t)blockIdx.z * g.M + m) * g.N + n] = acc[i][j];
      } else {
        double c = g.alpha * acc[i][j];
        if (g.beta != 0.0) c += g.beta * g.C[m * g.ldc + n];
        if (g.gamma != 0.0) c += g.gamma * g.D[m * g.ldd + n];
        if (g.delta != 0.0) c += g.delta * g.E[m * g.lde + n];
        g.C[m * g.ldc + n] = c;
      }
    }
}

template <Elt EA, Elt EB>
void launch_gemm(const GemmArgs& g, dim3 grid, cudaStream_t st) {
  TK_LAUNCH((k_dgemm<EA, EB>), grid, 256, 0, st, g);
}

constexpr int kSqBlocks = 296;
__global__ void k_sumsq_f32(const float* __restrict__ x, int64_t n, double* part) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[e];
    s += v * v;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
__global__ void k_sum_parts(const double* part, int n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += part[i];
    *out = s;
  }
}

}  // namespace

void dgemm(int64_t M, int64_t N, int64_t K, double alpha, MatRef A, MatRef B, double beta,
           double* C, int64_t ldc, double gamma, const double* D, int64_t ldd, DenseWs& ws,
           cudaStream_t st) {
  dgemm4(M, N, K, alpha, A, B, beta, C, ldc, gamma, D, ldd, 0.0, nullptr, 0, ws, st);
}

void dgemm4(int64_t M, int64_t N, int64_t K, double alpha, MatRef A, MatRef B, double beta,
            double* C, int64_t ldc, double gamma, const double* D, int64_t ldd, double delta,
            const double* E, int64_t lde, DenseWs& ws, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  GemmArgs g;
  g.M = M; g.N = N; g.K = K; g.A = A; g.B = B;
  g.alpha = alpha; g.beta = beta; g.gamma = gamma;
  g.C = C; g.ldc = ldc; g.D = D; g.ldd = ldd;
  g.delta = delta; g.E = E; g.lde = lde;
  const bool nn_fast = A.t == Elt::F64 && B.t == Elt::F64 && !A.trans && !B.trans && N <= 128 &&
                       M >= 64 && K > 0;
  if (nn_fast) {
    const int NC = (int)ceil_div(N, 32);
    const int64_t tiles_m = ceil_div(M, NBM);
    int64_t splits = 1;
    if (tiles_m < 148 && K > 4 * NBK)
      splits = std::max<int64_t>(1, std::min<int64_t>(ceil_div(148, tiles_m), ceil_div(K, 64)));
    g.kchunk = round_up(ceil_div(K, splits), NBK);
    splits = ceil_div(K, g.kchunk);
    if (splits > 1) {
      ws.splitk.ensure((size_t)(splits * M * N));
      g.part = ws.splitk.p;
    } else {
      g.part = nullptr;
    }
    const dim3 grid(1, (unsigned)tiles_m, (unsigned)splits);
    if (NC == 1) TK_LAUNCH(k_dgemm_nn<1>, grid, 256, 0, st, g);
    else if (NC == 2) TK_LAUNCH(k_dgemm_nn<2>, grid, 256, 0, st, g);
    else if (NC == 3) TK_LAUNCH(k_dgemm_nn<3>, grid, 256, 0, st, g);
    else TK_LAUNCH(k_dgemm_nn<4>, grid, 256, 0, st, g);
    if (splits > 1) {
      const int64_t blocks = std::min<int64_t>(ceil_div(M * N, 256), 148 * 8);
      TK_LAUNCH(k_splitk_reduce, (unsigned)blocks, 256, 0, st, M, N, (int)splits, ws.splitk.p,
                alpha, beta, C, ldc, gamma, D, ldd, delta, E, lde);
    }
    return;
  }
  const int64_t tiles = ceil_div(M, BM) * ceil_div(N, BN);
  int64_t splits = 1;
  if (K <= 0) {
    g.K = 0;
  } else if (tiles < 148 && K > 4 * BK) {
    splits = std::min<int64_t>(ceil_div(296, tiles), ceil_div(K, 64));
    if (splits < 1) splits = 1;
  }
  g.kchunk = K > 0 ? round_up(ceil_div(K, splits), BK) : BK;
  splits = K > 0 ? ceil_div(K, g.kchunk) : 1;
  if (splits > 1) {
    ws.splitk.ensure((size_t)(splits * M * N));
    g.part = ws.splitk.p;
  } else {
    g.part = nullptr;
  }
  dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, BM), (unsigned)splits);
#define TK_G(ea, eb) \
  if (A.t == ea && B.t == eb) launch_gemm<ea, eb>(g, grid, st); else
  TK_G(Elt::F64, Elt::F64) TK_G(Elt::SPLIT, Elt::F64) TK_G(Elt::F32, Elt::SPLIT)
  TK_G(Elt::F64, Elt::SPLIT) TK_G(Elt::F32, Elt::F64) TK_G(Elt::F64, Elt::F32)
  TK_G(Elt::SPLIT, Elt::SPLIT) TK_G(Elt::F32, Elt::F32) TK_G(Elt::SPLIT, Elt::F32)
  fail(TUCKER_E_ARG, "dgemm: operand types");
#undef TK_G
  if (splits > 1) {
    const int64_t blocks = std::min<int64_t>(ceil_div(M * N, 256), 148 * 8);
    TK_LAUNCH(k_splitk_reduce, (unsigned)blocks, 256, 0, st, M, N, (int)splits, ws.splitk.p,
              alpha, beta, C, ldc, gamma, D, ldd, delta, E, lde);
  }
}

double dnorm2_f32(const float* x, int64_t n, DenseWs& ws, cudaStream_t st) {
  ws.splitk.ensure(kSqBlocks + 1);
  TK_LAUNCH(k_sumsq_f32, kSqBlocks, 256, 0, st, x, n, ws.splitk.p);
  TK_LAUNCH(k_sum_parts, 1, 32, 0, st, ws.splitk.p, kSqBlocks, ws.splitk.p + kSqBlocks);
  double h = 0;
  TK_CUDA(cudaMemcpyAsync(&h, ws.splitk.p + kSqBlocks, sizeof(double), cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  return h;
}

}  // namespace tk
