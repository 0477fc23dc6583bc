// gram_tc.cu -- S = A A^T on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// Fig. 4 P:624-625 (S = Z_(n) Z_(n)^T) and Fig. 7/8 M_n = sum_s P_s P_s^T
// (= W W^T): both are SYRKs of a split-fp32 operand A (d x K, K contiguous).
//
// 3xTF32: a = hi + lo with hi = tf32(a), lo = tf32(a - hi) (spttmc.cu writes
// both), and a.b ~= hi.hi + hi.lo + lo.hi -- three kind::tf32 MMAs per K-step,
// fp32 accumulation in TMEM.  Every K-tile (32 products) the fp32 partial is
// drained from TMEM into fp64 registers (fp32 accumulation over the
// full K fails MP parity), double-buffered so the tensor core keeps running.
//
// CTA = one 128x128 upper-triangle tile (bi <= bj) x one K-split; warp roles:
//   warp 0      TMA producer (cp.async.bulk.tensor, 128B swizzle, 3-stage ring)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..9  epilogue: tcgen05.ld -> fp64 accumulate -> fp64 partial tile
// A second kernel sums the K-split partials in a fixed order (deterministic)
// and mirrors the tile into both triangles of S.
#include <cuda.h>

#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.cuh"
#include "tc_ptx.cuh"

namespace tk {
namespace {

constexpr int TM = 128;                 // tile rows (UMMA M)
constexpr int TN = 128;                 // tile cols (UMMA N)
constexpr int TKE = 32;                 // K elements per stage (128 B of fp32 -> one swizzle atom)
constexpr int STAGES = 3;
// K-tiles accumulated in fp32 in TMEM before each fp64 drain: 1 for short K
// (the drain is cheap there), DRAIN_LONG (128 products per fp32 partial) when a
// CTA streams many K-tiles and the drain would otherwise starve the tensor core
// (SURVEY F4 is about fp32 accumulation over the FULL K)
constexpr int DRAIN_LONG = 4;
constexpr int OPB = TM * TKE * 4;       // bytes of one operand tile (16 KB)
constexpr int STAGE_BYTES = 4 * OPB;    // A_hi, A_lo, B_hi, B_lo
constexpr int NUM_THREADS = 320;        // 10 warps
constexpr int TMEM_COLS = 256;          // two 128-column fp32 accumulators
constexpr uint32_t IDESC =
    (1u << 4) |               // D format: F32
    (2u << 7) | (2u << 10) |  // A, B format: TF32
    (0u << 15) | (0u << 16) | // A, B K-major
    ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);

using namespace tc;
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  tc::umma_tf32(tmem_d, a, b, IDESC, acc);
}

struct SyrkArgs {
  const int2* tiles;   // (bi, bj), bi <= bj
  int ntiles;
  int nkt;             // K-tiles in A
  int splits;          // split z takes the K-tiles z, z + splits, z + 2 splits, ...
  double* partial;     // [split][tile][128][128]
  int ktile;           // operand in the K-tile-major layout (3D tensor map: col, row, K-tile)
};

__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_syrk_tc(const __grid_constant__ CUtensorMap map_hi, const __grid_constant__ CUtensorMap map_lo,
              SyrkArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_slot;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x % p.ntiles;
  const int split = blockIdx.x / p.ntiles;
  const int2 bij = p.tiles[tile];
  const bool diag = bij.x == bij.y;
  // interleaved K-tiles: at any time all CTAs work inside a narrow K window, so
  // each operand panel streams from HBM about once and the re-reads by the
  // other tiles of its row block hit L2
  const int nk = split < p.nkt ? (p.nkt - split + p.splits - 1) / p.splits : 0;
  const int DRAIN = nk >= 64 ? DRAIN_LONG : 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 256);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      for (int i = 0; i < nk; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (uint32_t)((i / STAGES) & 1);
        mbar_wait(&empty_bar[s], ph ^ 1);
        uint8_t* st = smem + s * STAGE_BYTES;
        const int kt = split + i * p.splits;
        mbar_expect_tx(&full_bar[s], diag ? 2 * OPB : 4 * OPB);
        if (p.ktile) {  // rows past the operand's last row are zero-filled by TMA (out of bounds)
          tma_load_3d(st, &map_hi, &full_bar[s], 0, bij.x * TM, kt);
          tma_load_3d(st + OPB, &map_lo, &full_bar[s], 0, bij.x * TM, kt);
          if (!diag) {
            tma_load_3d(st + 2 * OPB, &map_hi, &full_bar[s], 0, bij.y * TM, kt);
            tma_load_3d(st + 3 * OPB, &map_lo, &full_bar[s], 0, bij.y * TM, kt);
          }
        } else {
          const int kcol = kt * TKE;
          tma_load_2d(st, &map_hi, &full_bar[s], kcol, bij.x * TM);
          tma_load_2d(st + OPB, &map_lo, &full_bar[s], kcol, bij.x * TM);
          if (!diag) {
            tma_load_2d(st + 2 * OPB, &map_hi, &full_bar[s], kcol, bij.y * TM);
            tma_load_2d(st + 3 * OPB, &map_lo, &full_bar[s], kcol, bij.y * TM);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      for (int i = 0; i < nk; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (uint32_t)((i / STAGES) & 1);
        const int grp = i / DRAIN, b = grp & 1;
        const bool first = (i % DRAIN) == 0, last = (i % DRAIN) == DRAIN - 1 || i == nk - 1;
        if (first) mbar_wait(&tempty_bar[b], (uint32_t)(((grp >> 1) & 1) ^ 1));
        mbar_wait(&full_bar[s], ph);
        tc_fence_after();
        const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
        const uint32_t ahi = base, alo = base + OPB;
        const uint32_t bhi = diag ? ahi : base + 2 * OPB, blo = diag ? alo : base + 3 * OPB;
        const uint32_t d = tmem_base + (uint32_t)(b * TN);
#pragma unroll
        for (int k = 0; k < TKE / 8; ++k) {
          const uint32_t off = (uint32_t)(k * 32);  // 8 tf32 = 32 bytes along K inside the atom
          umma_tf32(d, sw128_desc(ahi + off), sw128_desc(bhi + off), (k > 0 || !first) ? 1u : 0u);
          umma_tf32(d, sw128_desc(ahi + off), sw128_desc(blo + off), 1u);
          umma_tf32(d, sw128_desc(alo + off), sw128_desc(bhi + off), 1u);
        }
        umma_commit(&empty_bar[s]);         // smem stage free once these MMAs complete
        if (last) umma_commit(&tfull_bar[b]);  // fp32 partial of this K-tile group ready in TMEM
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int g = warp & 3;              // TMEM lane group this warp may access
    const int half = (warp - 2) >> 2;    // column half: 0 -> cols 0..63, 1 -> 64..127
    double acc[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) acc[j] = 0.0;
    const int ngrp = (nk + DRAIN - 1) / DRAIN;
    for (int grp = 0; grp < ngrp; ++grp) {
      const int b = grp & 1;
      mbar_wait(&tfull_bar[b], (uint32_t)((grp >> 1) & 1));
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(32 * g) << 16) + (uint32_t)(b * TN + 64 * half);
      float v0[32], v1[32];
      tmem_ld32(taddr, v0);
      tmem_ld32(taddr + 32, v1);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&tempty_bar[b]);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        acc[j] += (double)v0[j];
        acc[32 + j] += (double)v1[j];
      }
    }
    // fp64 partial tile: row = 32 g + lane, cols 64 half + j
    double* out = p.partial + ((int64_t)split * p.ntiles + tile) * (TM * TN) +
                  (int64_t)(32 * g + lane) * TN + 64 * half;
#pragma unroll
    for (int j = 0; j < 64; j += 2) *reinterpret_cast<double2*>(out + j) = make_double2(acc[j], acc[j + 1]);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
}

// S[i][j] = S[j][i] = sum_z partial[z][t][r][c] (fixed order); diagonal tiles r <= c only
__global__ void k_syrk_reduce(const double* __restrict__ partial, const int2* __restrict__ tiles,
                              int ntiles, int splits, int64_t d, double* __restrict__ S,
                              int64_t lds, const double* __restrict__ Sadd) {
  const int t = blockIdx.y;
  const int2 bij = tiles[t];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < TM * TN; e += gridDim.x * blockDim.x) {
    const int r = e / TN, c = e % TN;
    if (bij.x == bij.y && r > c) continue;
    const int64_t i = (int64_t)bij.x * TM + r, j = (int64_t)bij.y * TN + c;
    if (i >= d || j >= d) continue;
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += partial[((int64_t)z * ntiles + t) * (TM * TN) + e];
    if (Sadd) s += Sadd[i * lds + j];
    S[i * lds + j] = s;
    S[j * lds + i] = s;
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    TK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess)
      fail(TUCKER_E_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    fn = (EncodeTiledFn)p;
  }
  return fn;
}

// K-tile-major operand: dims (32 columns, ldr rows, nkt K-tiles); boxes of 32 x 128 x 1;
// rows >= ldr read as zero (out-of-bounds fill), so no padding rows are stored or read
CUtensorMap make_map_ktile(const float* base, int64_t ldr, int64_t nkt) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  const cuuint64_t gdim[3] = {(cuuint64_t)TKE, (cuuint64_t)ldr, (cuuint64_t)nkt};
  const cuuint64_t gstride[2] = {(cuuint64_t)(TKE * 4), (cuuint64_t)(ldr * TKE * 4)};
  const cuuint32_t box[3] = {(cuuint32_t)TKE, (cuuint32_t)TM, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, gdim, gstride,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(TUCKER_E_CUDA, "cuTensorMapEncodeTiled (3D) failed (" + std::to_string((int)r) + ")");
  return m;
}

CUtensorMap make_map(const float* base, int64_t rows_pad, int64_t ld, int64_t kext) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  const cuuint64_t gdim[2] = {(cuuint64_t)kext, (cuuint64_t)rows_pad};
  const cuuint64_t gstride[1] = {(cuuint64_t)(ld * 4)};
  const cuuint32_t box[2] = {(cuuint32_t)TKE, (cuuint32_t)TM};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, gdim, gstride,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(TUCKER_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

}  // namespace

void gram_syrk_tc(const Split& A, double* S, int64_t lds, GramWs& ws, cudaStream_t st, const double* Sadd) {
  const int smem_bytes = STAGES * STAGE_BYTES + 1024;
  smem_optin((const void*)k_syrk_tc, smem_bytes);
  const int64_t d = A.rows;
  const int64_t rows_pad = round_up(d, TM);
  if ((!A.ktile && A.ld % TKE != 0) || A.K() % TKE != 0)
    fail(TUCKER_E_ARG, "gram_syrk_tc: ld and K must be multiples of 32");
  const int nb = (int)(rows_pad / TM);
  const int ntiles = nb * (nb + 1) / 2;
  const int nkt = (int)(A.K() / TKE);
  std::vector<int2> tiles;
  tiles.reserve(ntiles);
  for (int i = 0; i < nb; ++i)
    for (int j = i; j < nb; ++j) tiles.push_back(make_int2(i, j));
  // K-splits: one wave of CTAs over the SMs (>= 4 K-tiles per CTA)
  int nsm = 148;
  {
    int dev = 0;
    TK_CUDA(cudaGetDevice(&dev));
    TK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  }
  nsm = std::max(1, nsm - g_sm_reserve);
  const int splits = (int)std::max<int64_t>(1, std::min<int64_t>(nsm / ntiles, nkt / 4));
  ws.scratch.ensure(sizeof(int2) * tiles.size());
  TK_CUDA(cudaMemcpyAsync(ws.scratch.p, tiles.data(), sizeof(int2) * tiles.size(),
                          cudaMemcpyHostToDevice, st));
  ws.partial.ensure((size_t)splits * ntiles * TM * TN);
  const CUtensorMap mhi = A.ktile ? make_map_ktile(A.hi, A.ld, nkt) : make_map(A.hi, rows_pad, A.ld, A.K());
  const CUtensorMap mlo = A.ktile ? make_map_ktile(A.lo, A.ld, nkt) : make_map(A.lo, rows_pad, A.ld, A.K());
  SyrkArgs a;
  a.tiles = (const int2*)ws.scratch.p;
  a.ntiles = ntiles;
  a.nkt = nkt;
  a.splits = splits;
  a.partial = ws.partial.p;
  a.ktile = A.ktile ? 1 : 0;
  TK_LAUNCH(k_syrk_tc, (unsigned)(ntiles * splits), NUM_THREADS, (size_t)smem_bytes, st, mhi, mlo, a);
  TK_LAUNCH(k_syrk_reduce, dim3(16, (unsigned)ntiles), 256, 0, st, (const double*)ws.partial.p,
            (const int2*)ws.scratch.p, ntiles, splits, d, S, lds, Sadd);
}

// Path selection: fp64 DMMA when the SYRK is small enough to afford fp64
// (<= 2e10 FMA, ~1 ms at the measured 37 TFLOP/s; all HOOI Grams of configs 1-4),
// 3xTF32 tcgen05 with fp64 drains for the large MP Grams.
void gram_syrk(const Split& A, double* S, int64_t lds, GramWs& ws, cudaStream_t st, const double* Sadd, double fma_hint) {
  if (A.K() == 0) {  // empty K shard: S = 0 (or Sadd)
    if (Sadd) {
      TK_CUDA(cudaMemcpy2DAsync(S, lds * sizeof(double), Sadd, lds * sizeof(double), A.rows * sizeof(double), A.rows,
                                cudaMemcpyDeviceToDevice, st));
    } else {
      for (int64_t i = 0; i < A.rows; ++i) TK_CUDA(cudaMemsetAsync(S + i * lds, 0, A.rows * sizeof(double), st));
    }
    return;
  }
  const double fma = fma_hint > 0 ? fma_hint : 0.5 * (double)A.rows * (double)(A.rows + 1) * (double)A.K();
  if (fma <= 2e10 || gram_mode() == 1) gram_syrk_dmma(A, S, lds, ws, st, Sadd);
  else gram_syrk_tc(A, S, lds, ws, st, Sadd);
}

int gram_path_id() { return gram_mode(); }

}  // namespace tk
