// gram_simt.cu -- fp64 SYRK paths, S = A A^T (A = hi + lo split fp32, so every
// product of two operand values is exact in fp64).  Fig. 4
// (Z_(n) Z_(n)^T) / Fig. 7 M_n.
//   * k_syrk_dmma: the fp64 tensor cores (mma.sync m8n8k4 f64 -> DMMA), 64x64
//     upper-triangle tiles x interleaved K splits, fixed-order split reduction.
//     Used for Grams small enough to afford fp64 (gram_syrk's threshold): the
//     bulk eigenvectors next to an outlier theta_1 >> theta_J are sensitive to
//     relative errors of S at the 1e-7 level that 3xTF32 leaves (config 4 HOOI,
//     theta_1 / gap ~ 1e4).
// (TUCKER_GRAM_FP64=1 sends every Gram through DMMA: a precision experiment switch,
// used to separate Gram rounding from projection rounding at config 5.)
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.cuh"

namespace tk {
namespace {

// ---------------------------------------------------------------- DMMA path --
constexpr int DT = 64, DKC = 32, DSP = DKC + 4;  // tile, K chunk, smem row stride (conflict-free)

__device__ __forceinline__ void dmma8(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// CTA = one 64x64 upper-triangle tile (bi <= bj) x one split (K chunks z, z +
// splits, ...); 8 warps, warp w owns tile rows 8w..8w+7 against all 8 column
// tiles.  Operands staged as fp64 (hi + lo) in shared memory.
// ktile: operand in the K-tile-major layout (lda = its row count, rows >= lda read as 0)
__global__ void __launch_bounds__(256) k_syrk_dmma(const float* __restrict__ hi, const float* __restrict__ lo,
                                                   int64_t lda, int nchunks, int ntiles, int splits,
                                                   const int2* __restrict__ tiles, double* __restrict__ part,
                                                   int ktile) {
  __shared__ double As[DT * DSP], Bs[DT * DSP];
  const int tile = blockIdx.x % ntiles, z = blockIdx.x / ntiles;
  const int2 bij = tiles[tile];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ar = lane >> 2, aq = lane & 3;
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
  const int64_t rstride = ktile ? DKC : lda;  // element (r, k): ktile (k / 32) 32 lda + 32 r + k % 32
  const float* hA = hi + (int64_t)bij.x * DT * rstride;
  const float* lA = lo + (int64_t)bij.x * DT * rstride;
  const float* hB = hi + (int64_t)bij.y * DT * rstride;
  const float* lB = lo + (int64_t)bij.y * DT * rstride;
  const int64_t ra = (int64_t)bij.x * DT, rb = (int64_t)bij.y * DT;
  // the next chunk's operands are prefetched into registers while the
  // current chunk's DMMAs run (one smem buffer); diagonal tiles load A only
  const bool diag = bij.x == bij.y;
  constexpr int PER = DT * DKC / 256;  // elements per thread per operand (8)
  float pah[PER], pal[PER], pbh[PER], pbl[PER];
  auto gload = [&](int ch) {
    const int k0 = ch * DKC;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = threadIdx.x + 256 * u, r = e >> 5, kk = e & 31;
      if (ktile) {
        const int64_t o = (int64_t)(k0 / DKC) * DKC * lda + (int64_t)r * DKC + kk;
        const bool va = ra + r < lda, vb = rb + r < lda;
        pah[u] = va ? __ldg(hA + o) : 0.f;
        pal[u] = va ? __ldg(lA + o) : 0.f;
        if (!diag) {
          pbh[u] = vb ? __ldg(hB + o) : 0.f;
          pbl[u] = vb ? __ldg(lB + o) : 0.f;
        }
      } else {
        const int64_t o = (int64_t)r * lda + k0 + kk;
        pah[u] = __ldg(hA + o);
        pal[u] = __ldg(lA + o);
        if (!diag) {
          pbh[u] = __ldg(hB + o);
          pbl[u] = __ldg(lB + o);
        }
      }
    }
  };
  if (z < nchunks) gload(z);
  const double* Bsrc = diag ? As : Bs;
  for (int ch = z; ch < nchunks; ch += splits) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = threadIdx.x + 256 * u, r = e >> 5, kk = e & 31;
      As[r * DSP + kk] = (double)pah[u] + (double)pal[u];
      if (!diag) Bs[r * DSP + kk] = (double)pbh[u] + (double)pbl[u];
    }
    __syncthreads();
    if (ch + splits < nchunks) gload(ch + splits);
    const double* ap = As + (8 * warp + ar) * DSP + aq;
    const double* bp = Bsrc + ar * DSP + aq;
#pragma unroll
    for (int kb = 0; kb < DKC; kb += 4) {
      const double a = ap[kb];
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma8(acc[j][0], acc[j][1], a, bp[8 * j * DSP + kb]);
    }
    __syncthreads();
  }
  double* out = part + ((size_t)z * ntiles + tile) * (DT * DT);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int r = 8 * warp + ar, c = 8 * j + 2 * aq;
    out[r * DT + c] = acc[j][0];
    out[r * DT + c + 1] = acc[j][1];
  }
}

// S[i][j] = S[j][i] = sum_z part[z][t][r][c] (fixed order); diagonal tiles r <= c only
__global__ void k_syrk_dmma_reduce(const double* __restrict__ part, const int2* __restrict__ tiles, int ntiles,
                                   int splits, int64_t d, double* __restrict__ S, int64_t lds,
                                   const double* __restrict__ Sadd) {
  const int t = blockIdx.y;
  const int2 bij = tiles[t];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < DT * DT; e += gridDim.x * blockDim.x) {
    const int r = e / DT, c = e % DT;
    if (bij.x == bij.y && r > c) continue;
    const int64_t i = (int64_t)bij.x * DT + r, j = (int64_t)bij.y * DT + c;
    if (i >= d || j >= d) continue;
    double s = 0.0;
    for (int q = 0; q < splits; ++q) s += part[((size_t)q * ntiles + t) * (DT * DT) + e];
    if (Sadd) s += Sadd[i * lds + j];
    S[i * lds + j] = s;
    S[j * lds + i] = s;
  }
}

}  // namespace

void gram_syrk_dmma(const Split& A, double* S, int64_t lds, GramWs& ws, cudaStream_t st, const double* Sadd) {
  const int64_t d = A.rows;
  const int nb = (int)ceil_div(d, DT);
  const int ntiles = nb * (nb + 1) / 2;
  if ((!A.ktile && A.ld % DKC != 0) || A.K() % DKC != 0)
    fail(TUCKER_E_ARG, "gram_syrk_dmma: ld and K must be multiples of 32");
  const int nchunks = (int)(A.K() / DKC);
  int nsm = 148;
  {
    int dev = 0;
    TK_CUDA(cudaGetDevice(&dev));
    TK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  }
  nsm = std::max(1, nsm - g_sm_reserve);
  // about two waves of 256-thread CTAs, >= 4 chunks per CTA
  const int splits = (int)std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(1, 2 * nsm / ntiles), nchunks / 4));
  std::vector<int2> tiles;
  tiles.reserve(ntiles);
  for (int i = 0; i < nb; ++i)
    for (int j = i; j < nb; ++j) tiles.push_back(make_int2(i, j));
  ws.scratch.ensure(sizeof(int2) * tiles.size());
  TK_CUDA(cudaMemcpyAsync(ws.scratch.p, tiles.data(), sizeof(int2) * tiles.size(), cudaMemcpyHostToDevice, st));
  ws.partial.ensure((size_t)splits * ntiles * DT * DT);
  TK_LAUNCH(k_syrk_dmma, (unsigned)(ntiles * splits), 256, 0, st, A.hi, A.lo, A.ld, nchunks, ntiles, splits,
            (const int2*)ws.scratch.p, ws.partial.p, A.ktile ? 1 : 0);
  TK_LAUNCH(k_syrk_dmma_reduce, dim3(8, (unsigned)ntiles), 256, 0, st, (const double*)ws.partial.p,
            (const int2*)ws.scratch.p, ntiles, splits, d, S, lds, Sadd);
}

int gram_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = std::getenv("TUCKER_GRAM_FP64");  // precision experiments: every Gram in fp64
    mode = (e && std::strcmp(e, "1") == 0) ? 1 : 0;
  }
  return mode;
}

}  // namespace tk
