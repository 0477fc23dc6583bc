// gram_simt.cu -- reference fp64 SIMT SYRK, S = A A^T (A = hi + lo split fp32).
// Used to validate the tcgen05 kernel (gram_tc.cu) and selectable with
// TUCKER_GRAM=simt.  Fig. 4 P:624-625 (Z_(n) Z_(n)^T) / Fig. 7 M_n.
#include <cstdlib>
#include <cstring>

#include "internal.cuh"

namespace tk {
namespace {

constexpr int TB = 64, TK = 16;

__global__ void __launch_bounds__(256) k_syrk_simt(const float* __restrict__ hi,
                                                   const float* __restrict__ lo, int64_t d,
                                                   int64_t K, int64_t lda, double* __restrict__ S,
                                                   int64_t lds) {
  // upper-triangle tile (bi <= bj) from a linear block index
  int64_t t = blockIdx.x, bi = 0;
  const int64_t nb = (d + TB - 1) / TB;
  while (t >= nb - bi) { t -= nb - bi; ++bi; }
  const int64_t bj = bi + t;
  __shared__ double As[TK][TB + 1], Bs[TK][TB + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  double acc[4][4] = {};
  for (int64_t k0 = 0; k0 < K; k0 += TK) {
    for (int e = tid; e < TB * TK; e += 256) {
      const int kk = e % TK, rr = e / TK;
      const int64_t k = k0 + kk;
      const int64_t ra = bi * TB + rr, rb = bj * TB + rr;
      As[kk][rr] = (ra < d && k < K) ? (double)hi[ra * lda + k] + (double)lo[ra * lda + k] : 0.0;
      Bs[kk][rr] = (rb < d && k < K) ? (double)hi[rb * lda + k] + (double)lo[rb * lda + k] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
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
      const int64_t r = bi * TB + ty + 16 * i, c = bj * TB + tx + 16 * j;
      if (r < d && c < d) {
        S[r * lds + c] = acc[i][j];
        S[c * lds + r] = acc[i][j];
      }
    }
}

}  // namespace

void gram_syrk_simt(const Split& A, double* S, int64_t lds, cudaStream_t st) {
  const int64_t nb = ceil_div(A.rows, TB);
  TK_LAUNCH(k_syrk_simt, (unsigned)(nb * (nb + 1) / 2), 256, 0, st, A.hi, A.lo, A.rows, A.cols,
            A.ld, S, lds);
}

int gram_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = std::getenv("TUCKER_GRAM");
    mode = (e && std::strcmp(e, "simt") == 0) ? 1 : 0;
  }
  return mode;
}

}  // namespace tk
