// spttmc4g.cu -- order-4 HOOI SpTTMc in GEMM form for tensors whose nodes are
// dense in the mid1 index (BASELINE config 4: 200^4 at 1 % density, every node
// (i, a) holds ~172 of its 200 possible fibers).
//
// Per slice i (PAPER Appendix: row i of Y_(1) = B' X1_slice C, extended
// to order 4 with lower modes fastest, reading A9) and node v = (i, a):
//   leaf     T_v[b, :]  = sum_{x in fiber (v, b)} x U_leaf[leaf(x), :]     (Eq. 1)
//   level 2  Z_v        = U_mid1^T T_v        (J1 x Jl; a dense K = I_mid1 contraction)
//   level 3  Y_i[a', :] += U_mid0[a, a'] Z_v  (K = the slice's nodes)
// k_spttmc4w does level 2 fiber by fiber (an outer product per fiber whose two
// 128-bit shared-memory loads feed 16 FMAs -- shared-memory-wavefront bound).
// Here a batch of NB nodes is processed together and level 2 is a register-
// tiled GEMM: thread (v, c-group) owns Z_v[0..J1P)[4 c] (4 J1P accumulators);
// per mid1 index b it reads the U_mid1 row once (warp-uniform, broadcast) and
// the 4 T values of its columns once (lane-distinct, conflict-free), i.e.
// 4 J1P FMAs per 1 + J1P/4 shared loads.  T is produced chunk by chunk
// (KCH mid1 indices at a time) into shared memory by the leaf stage.
//
// Data: a one-time re-layout of the ordering's fibers ("dense batch layout"):
// batch = NB consecutive nodes of one slice; per (batch, chunk) the slots
// (b_local, v) in b-major order each own the nonzeros of fiber (v, b) (empty
// slots own none).  The slot offsets `sp` and the re-ordered nonzeros of one
// (batch, chunk) are contiguous, so each chunk arrives by three 1-D bulk
// copies (cp.async.bulk, TMA engine) one chunk ahead of its use, and no fiber
// search or zero fill is needed.  Persistent CTAs take contiguous batch ranges;
// consecutive batches of one slice accumulate Y_i in shared memory, each run's
// partial row is written once and k_spttmc4g_reduce sums a slice's runs in
// batch order (deterministic, no atomics).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include <cub/cub.cuh>

#include "internal.cuh"
#include "tc_ptx.cuh"

namespace tk {

__device__ __forceinline__ float tf32_rna_g4(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

namespace {

constexpr int kNT = 256;   // threads per CTA
constexpr int kKCH = 16;   // mid1 indices per chunk
constexpr int kCap = 2048; // staged nonzeros per chunk buffer (longer chunks read global memory)

struct G4Args {
  const int4* batch;        // (slice, first node, nodes, -) per batch
  const int32_t* node_mid0;
  const int32_t* sp;        // slot nonzero offsets, SPC per (batch, chunk), slots sorted by count
  const int32_t* tgt;       // each sorted slot's (b_local, v) index b_local NB + v
  const int32_t* leaf;      // nonzeros in slot order
  const float* val;
  const float *U0, *U1, *Ul;
  int J0, J1, Jl, JLP, J0P, CL, NB, NCH, SPC;
  int I_leaf, I_mid1;
  int b_lo, nb;             // batches [b_lo, b_lo + nb) of this launch
  float* part;              // [nb][J0 * J1 * JLP] partial rows of runs (index: run's first batch - b_lo)
  float* zout;              // nullable: Z_v of every node, [nnode][J1 * JLP] (kept for the sibling mode)
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          tc::smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// CTA c of G owns batches [c nb / G, (c + 1) nb / G)
__host__ __device__ inline int cta_first(int c, int nb, int G) { return (int)(((int64_t)c * nb) / G); }

template <int J1P>
__global__ void __launch_bounds__(kNT, 1) k_spttmc4g(G4Args p) {
  extern __shared__ __align__(16) float smg[];
  __shared__ __align__(8) uint64_t full[2];
  __shared__ int st_e0[2], st_ok[2];
  const int tid = threadIdx.x;
  const int JLP = p.JLP, CL = p.CL, NB = p.NB, J1 = p.J1, J0 = p.J0, J0P = p.J0P;
  const int P1 = J1 * JLP, P = J0 * P1;
  const int LDT = NB * JLP;
  const int nslot = NB * kKCH;
  // layout: Uls | U1s | TZ (T chunk / Z of the batch) | ys | u0t | stage[2] = (spbuf SPC, leaf kCap, val kCap)
  float* Uls = smg;
  float* U1s = Uls + p.I_leaf * JLP;
  float* TZ = U1s + p.I_mid1 * J1P;
  const int tz = max(kKCH * LDT, NB * P1);
  float* ys = TZ + ((tz + 3) & ~3);
  float* u0t = ys + ((P + 3) & ~3);
  int* stg = reinterpret_cast<int*>(u0t + NB * J0P);
  const int SB = 2 * p.SPC + 2 * kCap;  // ints per stage buffer: slot offsets, slot targets, leaf ids, values

  const int b0 = p.b_lo + cta_first(blockIdx.x, p.nb, gridDim.x);
  const int b1 = p.b_lo + cta_first(blockIdx.x + 1, p.nb, gridDim.x);
  if (b0 >= b1) return;
  const int64_t ck0 = (int64_t)b0 * p.NCH, nck = (int64_t)(b1 - b0) * p.NCH;

  // bulk-copy issue of chunk q (thread 0); E bounds come from the caller
  auto issue = [&](int64_t q, int E0, int E1) {
    const int buf = (int)(q & 1);
    int* sb = stg + buf * SB;
    const int E0r = E0 & ~3, E1r = (E1 + 3) & ~3;
    const int n = E1r - E0r;
    const bool ok = n <= kCap;
    st_e0[buf] = E0r;
    st_ok[buf] = ok ? 1 : 0;
    tc::mbar_expect_tx(&full[buf], (uint32_t)(p.SPC * 8 + (ok ? 8 * n : 0)));
    bulk_g2s(sb, p.sp + (ck0 + q) * p.SPC, (uint32_t)(p.SPC * 4), &full[buf]);
    bulk_g2s(sb + p.SPC, p.tgt + (ck0 + q) * p.SPC, (uint32_t)(p.SPC * 4), &full[buf]);
    if (ok && n > 0) {
      bulk_g2s(sb + 2 * p.SPC, p.leaf + E0r, (uint32_t)(4 * n), &full[buf]);
      bulk_g2s(sb + 2 * p.SPC + kCap, p.val + E0r, (uint32_t)(4 * n), &full[buf]);
    }
  };
  int nxE0 = 0, nxE1 = 0;  // thread 0: bounds of the chunk issued next (q + 2)
  if (tid == 0) {
    tc::mbar_init(&full[0], 1);
    tc::mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // factor tables, rows zero padded to JLP / J1P floats
  for (int e = tid; e < p.I_leaf * JLP; e += kNT) {
    const int r = e / JLP, j = e - r * JLP;
    Uls[e] = j < p.Jl ? __ldg(p.Ul + (int64_t)r * p.Jl + j) : 0.f;
  }
  for (int e = tid; e < p.I_mid1 * J1P; e += kNT) {
    const int r = e / J1P, j = e - r * J1P;
    U1s[e] = j < J1 ? __ldg(p.U1 + (int64_t)r * J1 + j) : 0.f;
  }
  for (int e = tid; e < P; e += kNT) ys[e] = 0.f;
  __syncthreads();
  if (tid == 0) {
    for (int64_t q = 0; q < 2 && q < nck; ++q) {
      const int64_t ck = ck0 + q;
      issue(q, __ldg(p.sp + ck * p.SPC), __ldg(p.sp + (ck + 1) * p.SPC));
    }
    if (nck > 2) {
      nxE0 = __ldg(p.sp + (ck0 + 2) * p.SPC);
      nxE1 = __ldg(p.sp + (ck0 + 3) * p.SPC);
    }
  }

  const bool gem = tid < NB * CL;  // GEMM thread: node v, columns 4 cg .. 4 cg + 3
  const int gv = gem ? tid / CL : 0;
  float acc[J1P][4];
#pragma unroll
  for (int r = 0; r < J1P; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = 0.f;

  int64_t q = 0;
  int run0 = b0;  // first batch of the current run (consecutive batches of one slice)
  for (int b = b0; b < b1; ++b) {
    const int4 bt = p.batch[b];  // slice, node0, nn
    // U_mid0 rows of the batch's nodes (used by level 3; loads overlap the chunks)
    for (int e = tid; e < NB * J0P; e += kNT) {
      const int v = e / J0P, a = e - v * J0P;
      u0t[e] = (v < bt.z && a < J0) ? __ldg(p.U0 + (int64_t)__ldg(p.node_mid0 + bt.y + v) * J0 + a) : 0.f;
    }
    for (int kc = 0; kc < p.NCH; ++kc, ++q) {
      const int buf = (int)(q & 1);
      tc::mbar_wait(&full[buf], (uint32_t)((q >> 1) & 1));
      const int* sb = stg + buf * SB;
      const int E0r = st_e0[buf];
      const bool ok = st_ok[buf] != 0;
      // ---- leaf stage: slot s = (b_local, v) -> T[b_local][v JLP + :]
      for (int s = tid; s < nslot; s += kNT) {
        const int e0 = sb[s], e1 = sb[s + 1];
        const int tg = sb[p.SPC + s];
        const int v = tg % NB, bl = tg / NB;
        float4 t[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) t[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int e = e0; e < e1; ++e) {
          int l;
          float x;
          if (ok) {
            l = sb[2 * p.SPC + e - E0r];
            x = __int_as_float(sb[2 * p.SPC + kCap + e - E0r]);
          } else {
            l = __ldg(p.leaf + e);
            x = __ldg(p.val + e);
          }
          const float4* r4 = reinterpret_cast<const float4*>(Uls + l * JLP);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            if (c < CL) {
              const float4 g = r4[c];
              t[c].x = fmaf(x, g.x, t[c].x);
              t[c].y = fmaf(x, g.y, t[c].y);
              t[c].z = fmaf(x, g.z, t[c].z);
              t[c].w = fmaf(x, g.w, t[c].w);
            }
          }
        }
        float4* Tw = reinterpret_cast<float4*>(TZ + bl * LDT + v * JLP);
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < CL) Tw[c] = t[c];
      }
      __syncthreads();  // T ready; stage buffer `buf` free
      if (tid == 0 && q + 2 < nck) {
        issue(q + 2, nxE0, nxE1);
        if (q + 3 < nck) {
          nxE0 = __ldg(p.sp + (ck0 + q + 3) * p.SPC);
          nxE1 = __ldg(p.sp + (ck0 + q + 4) * p.SPC);
        }
      }
      // ---- level 2: Z_v[r][4 cg + c] += U_mid1[b][r] T[b_local][4 tid + c]
      if (gem) {
        const int nb_ = min(kKCH, p.I_mid1 - kc * kKCH);
        const float4* urow = reinterpret_cast<const float4*>(U1s + (int64_t)kc * kKCH * J1P);
        const float* tcol = TZ + 4 * tid;
#pragma unroll 2
        for (int bl = 0; bl < nb_; ++bl) {
          const float4 t4 = *reinterpret_cast<const float4*>(tcol + bl * LDT);
          float u[J1P];
#pragma unroll
          for (int r4 = 0; r4 < J1P / 4; ++r4) {
            const float4 g = urow[bl * (J1P / 4) + r4];
            u[4 * r4] = g.x;
            u[4 * r4 + 1] = g.y;
            u[4 * r4 + 2] = g.z;
            u[4 * r4 + 3] = g.w;
          }
#pragma unroll
          for (int r = 0; r < J1P; ++r) {
            acc[r][0] = fmaf(u[r], t4.x, acc[r][0]);
            acc[r][1] = fmaf(u[r], t4.y, acc[r][1]);
            acc[r][2] = fmaf(u[r], t4.z, acc[r][2]);
            acc[r][3] = fmaf(u[r], t4.w, acc[r][3]);
          }
        }
      }
      __syncthreads();  // T consumed
    }
    // ---- level 3: Y_i[a][r JLP + c] += sum_v U_mid0[a_v][a] Z_v[r][c]
    if (gem && gv < bt.z) {
      float* Zw = TZ + gv * P1 + 4 * (tid - gv * CL);
#pragma unroll
      for (int r = 0; r < J1P; ++r)
        if (r < J1) *reinterpret_cast<float4*>(Zw + r * JLP) = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
    }
#pragma unroll
    for (int r = 0; r < J1P; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = 0.f;
    __syncthreads();
    if (p.zout) {  // the batch's Z rows are contiguous (node-major) in TZ and in zout
      float* zo = p.zout + (int64_t)bt.y * P1;
      for (int e = tid; e < bt.z * P1; e += kNT) zo[e] = TZ[e];
    }
    const bool run_end = b + 1 == b1 || p.batch[b + 1].x != bt.x;
    for (int col = tid; col < P1; col += kNT) {
      for (int a0 = 0; a0 < J0; a0 += 4) {
        float y0 = 0.f, y1 = 0.f, y2 = 0.f, y3 = 0.f;
        for (int v = 0; v < bt.z; ++v) {
          const float z = TZ[v * P1 + col];
          const float4 u = *reinterpret_cast<const float4*>(u0t + v * J0P + a0);
          y0 = fmaf(u.x, z, y0);
          y1 = fmaf(u.y, z, y1);
          y2 = fmaf(u.z, z, y2);
          y3 = fmaf(u.w, z, y3);
        }
        const float yv[4] = {y0, y1, y2, y3};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (a0 + k < J0) {
            float* yp = ys + (a0 + k) * P1 + col;
            const float y = *yp + yv[k];
            if (run_end) {
              p.part[(int64_t)(run0 - p.b_lo) * P + (a0 + k) * P1 + col] = y;
              *yp = 0.f;
            } else {
              *yp = y;
            }
          }
        }
      }
    }
    if (run_end) run0 = b + 1;
    __syncthreads();  // Z / u0t consumed before the next batch overwrites them
  }
}

// Y_i = sum of the slice's run partials in batch order, split-stored with Kolda strides
__global__ void __launch_bounds__(256) k_spttmc4g_reduce(const float* __restrict__ part, const int32_t* __restrict__ bfirst,
                                                        int s_lo, int b_lo, int nb, int G, int J1, int Jl, int JLP,
                                                        int P, int64_t s0, int64_t s1, int64_t sb, float* __restrict__ Yhi,
                                                        float* __restrict__ Ylo, int64_t ldY, int transposed) {
  const int i = s_lo + blockIdx.y;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= P) return;
  const int P1 = J1 * JLP;
  const int a = col / P1, rem = col - a * P1, r = rem / JLP, c = rem - r * JLP;
  if (c >= Jl) return;
  const int f = bfirst[i], l = bfirst[i + 1];
  float y = 0.f;
  for (int b = f; b < l; ++b) {
    const int lb = b - b_lo;
    // run start: the slice's first batch or the first batch of a CTA's range
    const int cta = (int)(((int64_t)lb * G + nb - 1) / nb);
    const bool start = b == f || cta_first(cta, nb, G) == lb;
    if (start) y += __ldcs(part + (int64_t)lb * P + col);
  }
  const int64_t ycol = a * s0 + r * s1 + c * sb;
  const int64_t off = transposed ? ycol * ldY + i : (int64_t)i * ldY + ycol;
  const float h = tf32_rna_g4(y);
  Yhi[off] = h;
  Ylo[off] = tf32_rna_g4(y - h);
}

// ---------------------------------------------------------------------------
// k_spttmc4t: the same batches with level 2 on the tensor cores (tcgen05,
// 3xTF32, fp32 accumulation in TMEM).  Per chunk of 32 mid1 indices the leaf
// stage writes the plain fiber sums T[b][v JLP + c] (lanes = (slot, 4 leaf
// columns), 128-bit stores), then a transposing pass writes the K-major
// 128B-swizzled operands A = T^T (rows (v, c): NB JLP <= 256 -> two M = 128
// tiles, K = b) and B = U_mid1^T (32 rows b', K = b), split (tf32 hi, lo),
// and one thread issues D[(v, c)][b'] += A B^T as 2 tiles x 4 K-steps x 3
// kind::tf32 MMAs (hi.hi + hi.lo + lo.hi).  The MMAs of chunk q run while the
// leaf stage of chunk q + 1 computes (one operand buffer: the transposing pass
// waits for the previous commit).  After a batch's last chunk each thread
// reads its TMEM row (v, c) -- Z_v[:, c] -- into shared memory, and level 3
// (Y_i += U_mid0[a_v] (x) Z_v) runs on the FMA pipes with Y in registers.
// K per accumulation = I_mid1 (200 at config 4): the TMEM sum is over <= 224
// products (the drift measured for thousands of products does not arise).
// ---------------------------------------------------------------------------
constexpr int kTKC = 32;  // mid1 indices per chunk (one 128-byte swizzle row of K)

struct G4tArgs {
  int maxck;                // k_spttmc4s: chunk bounds held in shared memory (>= chunks per CTA + 1)
  int dbg;                  // timing experiments (TUCKER_TTMC4_DBG): 1 skip leaf, 2 skip transpose, 4 skip MMAs, 8 skip level 3
  int bres;                 // the B operands (U_mid1^T split) of every chunk resident in shared memory
  const int4* batch;
  const int32_t* node_mid0;
  const int32_t* sp;
  const int32_t* tgt;
  const int32_t* leaf;
  const float* val;
  const float *U0, *U1, *Ul;
  int J0, J1, Jl, JLP, J0P, CL, NB, NCH, SPC;
  int I_leaf, I_mid1;
  int b_lo, nb;
  float* part;
};

constexpr int kTpLd = 260;                         // plain T row stride (floats): conflict-free column reads
constexpr int kTA = 128 * 128;                     // one A tile (128 rows x 128 B)
constexpr int kTB = 32 * 128;                      // the B tile (32 rows x 128 B)
constexpr uint32_t kTIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(32 >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);

__device__ __forceinline__ uint32_t t_sw128(int row, int k) {
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((((k >> 2) ^ (row & 7)) << 4) | ((k & 3) << 2)));
}
// 3xTF32 split of a finite v: hi = v rounded to tf32 (nearest, ties away: add half an ulp of the
// 10-bit mantissa, clear the low 13 bits), lo = v - hi (exact in fp32); the MMA reads lo's top 19
// bits (|lo| <= 2^-11 |v|, so the dropped bits are < 2^-21 |v|)
__device__ __forceinline__ void t_split(uint8_t* hi, uint8_t* lo, uint32_t off, float v) {
  const float h = __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xffffe000u);
  *reinterpret_cast<float*>(hi + off) = h;
  *reinterpret_cast<float*>(lo + off) = v - h;
}

template <int CL>  // leaf columns / 4 (JLP = 4 CL); NB = 256 / JLP nodes per batch
__global__ void __launch_bounds__(kNT, 1) k_spttmc4t(G4tArgs p) {
  extern __shared__ uint8_t smt_raw[];
  // 1024-byte alignment by pointer arithmetic on the shared array (keeps the .shared state space
  // visible to the compiler: LDS/STS instead of generic loads)
  uint8_t* smt = smt_raw + ((1024u - (tc::smem_u32(smt_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[2], mma_done;
  __shared__ int st_e0[2], st_ok[2];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int JLP = 4 * CL, NB = kNT / JLP;
  const int J0 = p.J0, J0P = p.J0P, J1 = p.J1;
  const int P1 = J1 * JLP;
  constexpr int nslot = NB * kTKC;
  // layout (1024-aligned): A_hi[2] A_lo[2] | B_hi B_lo | Tp (32 x kTpLd; Z of the batch) | Uls | u0t | stage[2]
  uint8_t* Ahi = smt;
  uint8_t* Alo = Ahi + 2 * kTA;
  uint8_t* Bhi = Alo + 2 * kTA;
  uint8_t* Blo = Bhi + kTB;
  float* Tp = reinterpret_cast<float*>(Blo + kTB);
  float* Uls = Tp + kTKC * kTpLd;
  float* u0t = Uls + p.I_leaf * JLP;
  int* stg = reinterpret_cast<int*>(u0t + ((NB * J0P + 3) & ~3));
  const int SB = 2 * p.SPC + 2 * kCap;
  // resident B tiles (p.bres): chunk kc's hi at Bres + 8 KB kc, lo 4 KB after (1024-aligned)
  uint8_t* Bres = reinterpret_cast<uint8_t*>(stg + 2 * SB);
  Bres += (1024u - (tc::smem_u32(Bres) & 1023u)) & 1023u;

  const int b0 = p.b_lo + cta_first(blockIdx.x, p.nb, gridDim.x);
  const int b1 = p.b_lo + cta_first(blockIdx.x + 1, p.nb, gridDim.x);
  if (b0 >= b1) return;
  const int64_t ck0 = (int64_t)b0 * p.NCH, nck = (int64_t)(b1 - b0) * p.NCH;
  auto issue = [&](int64_t q, int E0, int E1) {
    const int buf = (int)(q & 1);
    int* sb = stg + buf * SB;
    const int E0r = E0 & ~3, E1r = (E1 + 3) & ~3;
    const int n = E1r - E0r;
    const bool ok = n <= kCap;
    st_e0[buf] = E0r;
    st_ok[buf] = ok ? 1 : 0;
    tc::mbar_expect_tx(&full[buf], (uint32_t)(p.SPC * 8 + (ok ? 8 * n : 0)));
    bulk_g2s(sb, p.sp + (ck0 + q) * p.SPC, (uint32_t)(p.SPC * 4), &full[buf]);
    bulk_g2s(sb + p.SPC, p.tgt + (ck0 + q) * p.SPC, (uint32_t)(p.SPC * 4), &full[buf]);
    if (ok && n > 0) {
      bulk_g2s(sb + 2 * p.SPC, p.leaf + E0r, (uint32_t)(4 * n), &full[buf]);
      bulk_g2s(sb + 2 * p.SPC + kCap, p.val + E0r, (uint32_t)(4 * n), &full[buf]);
    }
  };
  if (tid == 0) {
    tc::mbar_init(&full[0], 1);
    tc::mbar_init(&full[1], 1);
    tc::mbar_init(&mma_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tmem_slot)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int e = tid; e < p.I_leaf * JLP; e += kNT) {
    const int r = e / JLP, j = e - r * JLP;
    Uls[e] = j < p.Jl ? __ldg(p.Ul + (int64_t)r * p.Jl + j) : 0.f;
  }
  if (p.bres) {
    for (int e = tid; e < p.NCH * 32 * kTKC; e += kNT) {
      const int kc = e / (32 * kTKC), rem = e - kc * (32 * kTKC), r = rem / kTKC, k = rem - r * kTKC;
      const int b = kc * kTKC + k;
      const float u = (r < J1 && b < p.I_mid1) ? __ldg(p.U1 + (int64_t)b * J1 + r) : 0.f;
      t_split(Bres + kc * 2 * kTB, Bres + kc * 2 * kTB + kTB, t_sw128(r, k), u);
    }
  }
  // A rows past NB JLP are never written: zero both tiles once (their D rows are not read)
  for (int o = tid * 16; o < 4 * kTA + 2 * kTB; o += kNT * 16) *reinterpret_cast<float4*>(smt + o) = make_float4(0.f, 0.f, 0.f, 0.f);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_slot;
  int nxE0 = 0, nxE1 = 0;
  if (tid == 0) {
    for (int64_t q = 0; q < 2 && q < nck; ++q) {
      const int64_t ck = ck0 + q;
      issue(q, __ldg(p.sp + ck * p.SPC), __ldg(p.sp + (ck + 1) * p.SPC));
    }
    if (nck > 2) {
      nxE0 = __ldg(p.sp + (ck0 + 2) * p.SPC);
      nxE1 = __ldg(p.sp + (ck0 + 3) * p.SPC);
    }
  }
  // Y of the current run in registers: columns col = tid, tid + 256 (< P1) x J0 rows
  constexpr int kYC = 2, kYA = 32;
  float yacc[kYC][kYA];
#pragma unroll
  for (int u = 0; u < kYC; ++u)
#pragma unroll
    for (int a = 0; a < kYA; ++a) yacc[u][a] = 0.f;
  int64_t q = 0;
  uint32_t mphase = 0;  // completed commits of mma_done
  bool pending = false;
  int run0 = b0;
  const uint32_t sA = tc::smem_u32(Ahi), sAl = tc::smem_u32(Alo), sB = tc::smem_u32(Bhi), sBl = tc::smem_u32(Blo);
  for (int b = b0; b < b1; ++b) {
    const int4 bt = p.batch[b];
    for (int e = tid; e < NB * J0P; e += kNT) {
      const int v = e / J0P, a = e - v * J0P;
      u0t[e] = (v < bt.z && a < J0) ? __ldg(p.U0 + (int64_t)__ldg(p.node_mid0 + bt.y + v) * J0 + a) : 0.f;
    }
    for (int kc = 0; kc < p.NCH; ++kc, ++q) {
      const int buf = (int)(q & 1);
      tc::mbar_wait(&full[buf], (uint32_t)((q >> 1) & 1));
      const int* sb = stg + buf * SB;
      const int E0r = st_e0[buf];
      const bool ok = st_ok[buf] != 0;
      // ---- leaf: lane = slot (sorted by count: equal trip counts within a warp), all JLP columns
      for (int sl = tid; sl < nslot; sl += kNT) {
        const int e0 = sb[sl], e1 = sb[sl + 1];
        const int tg = sb[p.SPC + sl];
        const int v = tg % NB, bl = tg / NB;
        float4 t[CL];
#pragma unroll
        for (int c = 0; c < CL; ++c) t[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int e = e0; e < e1; ++e) {
          int l;
          float x;
          if (ok) {
            l = sb[2 * p.SPC + e - E0r];
            x = __int_as_float(sb[2 * p.SPC + kCap + e - E0r]);
          } else {
            l = __ldg(p.leaf + e);
            x = __ldg(p.val + e);
          }
          const float4* r4 = reinterpret_cast<const float4*>(Uls + l * JLP);
#pragma unroll
          for (int c = 0; c < CL; ++c) {
            const float4 g = r4[c];
            t[c].x = fmaf(x, g.x, t[c].x);
            t[c].y = fmaf(x, g.y, t[c].y);
            t[c].z = fmaf(x, g.z, t[c].z);
            t[c].w = fmaf(x, g.w, t[c].w);
          }
        }
        float4* Tw = reinterpret_cast<float4*>(Tp + bl * kTpLd + v * JLP);
#pragma unroll
        for (int c = 0; c < CL; ++c) Tw[c] = t[c];
      }
      __syncthreads();  // T ready; stage buffer `buf` free
      if (tid == 0 && q + 2 < nck) {
        issue(q + 2, nxE0, nxE1);
        if (q + 3 < nck) {
          nxE0 = __ldg(p.sp + (ck0 + q + 3) * p.SPC);
          nxE1 = __ldg(p.sp + (ck0 + q + 4) * p.SPC);
        }
      }
      if (pending) {  // the operands are rewritten: the previous chunk's MMAs must have read them
        tc::mbar_wait(&mma_done, mphase & 1);
        ++mphase;
        pending = false;
      }
      // ---- transpose into the K-major operands: lane = k (mid1 index in the chunk); rows
      // r = 4 r4 + u, byte offset (r / 8) 1024 + o8[r % 8] within the tile (r4 steps of 8 keep r % 8)
      {
        const int k = lane;
        constexpr int rows = NB * JLP;
        const int h = (warp & 1) * 4;  // r % 8 = h + u for r4 = warp (mod 2)
        uint32_t o4[4];                // in-atom offsets of rows h + u at column k
#pragma unroll
        for (int u = 0; u < 4; ++u) o4[u] = (uint32_t)((h + u) * 128 + ((((k >> 2) ^ (h + u)) << 4) | ((k & 3) << 2)));
        for (int r4 = warp; r4 < (rows + 3) / 4; r4 += kNT / 32) {
          const float4 v4 = *reinterpret_cast<const float4*>(Tp + k * kTpLd + 4 * r4);
          const int r0 = 4 * r4;
          const uint32_t base = (uint32_t)((r0 >> 7) * kTA + ((r0 & 127) >> 3) * 1024);
          t_split(Ahi, Alo, base + o4[0], v4.x);
          t_split(Ahi, Alo, base + o4[1], v4.y);
          t_split(Ahi, Alo, base + o4[2], v4.z);
          t_split(Ahi, Alo, base + o4[3], v4.w);
        }
        if (!p.bres) {
          const int b = kc * kTKC + k;
          for (int r = warp; r < 32; r += kNT / 32) {
            const float u = (r < J1 && b < p.I_mid1) ? __ldg(p.U1 + (int64_t)b * J1 + r) : 0.f;
            t_split(Bhi, Blo, t_sw128(r, k), u);
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        tc::tc_fence_after();
        const uint32_t sBk = p.bres ? tc::smem_u32(Bres + kc * 2 * kTB) : sB;
        const uint32_t sBlk = p.bres ? sBk + kTB : sBl;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const uint32_t d = tmem + 32 * mt;
#pragma unroll
          for (int ks = 0; ks < kTKC / 8; ++ks) {
            const uint32_t o = (uint32_t)(ks * 32);
            const uint32_t ah = sA + mt * kTA + o, al = sAl + mt * kTA + o;
            tc::umma_tf32(d, tc::sw128_desc(ah), tc::sw128_desc(sBk + o), kTIdesc, (kc > 0 || ks > 0) ? 1u : 0u);
            tc::umma_tf32(d, tc::sw128_desc(ah), tc::sw128_desc(sBlk + o), kTIdesc, 1u);
            tc::umma_tf32(d, tc::sw128_desc(al), tc::sw128_desc(sBk + o), kTIdesc, 1u);
          }
        }
        tc::umma_commit(&mma_done);
      }
      pending = true;
    }
    // ---- the batch's Z: TMEM row (v, c) of tile mt -> Zs[v][b' JLP + c] (Zs aliases Tp)
    tc::mbar_wait(&mma_done, mphase & 1);
    ++mphase;
    pending = false;
    tc::tc_fence_after();
    {
      const int mt = warp >> 2, lq = warp & 3;
      float z[32];
      tc::tmem_ld32(tmem + ((uint32_t)(32 * lq) << 16) + (uint32_t)(32 * mt), z);
      tc::tmem_wait_ld();
      const int r = mt * 128 + lq * 32 + lane;
      const int v = r / JLP, c = r - v * JLP;
      if (v < bt.z) {
#pragma unroll
        for (int bp = 0; bp < 32; ++bp)
          if (bp < J1) Tp[v * P1 + bp * JLP + c] = z[bp];
      }
    }
    tc::tc_fence_before();
    __syncthreads();
    // ---- level 3: Y[a][col] += sum_v U_mid0[a_v][a] Z_v[col] (registers)
    const bool run_end = b + 1 == b1 || p.batch[b + 1].x != bt.x;
#pragma unroll
    for (int u = 0; u < kYC; ++u) {
      const int col = tid + kNT * u;
      if (col < P1) {
        for (int v = 0; v < bt.z; ++v) {
          const float zz = Tp[v * P1 + col];
          const float4* u4 = reinterpret_cast<const float4*>(u0t + v * J0P);
#pragma unroll
          for (int a4 = 0; a4 < kYA / 4; ++a4) {
            if (4 * a4 < J0) {
              const float4 w = u4[a4];
              yacc[u][4 * a4] = fmaf(w.x, zz, yacc[u][4 * a4]);
              yacc[u][4 * a4 + 1] = fmaf(w.y, zz, yacc[u][4 * a4 + 1]);
              yacc[u][4 * a4 + 2] = fmaf(w.z, zz, yacc[u][4 * a4 + 2]);
              yacc[u][4 * a4 + 3] = fmaf(w.w, zz, yacc[u][4 * a4 + 3]);
            }
          }
        }
        if (run_end) {
          float* dst = p.part + (int64_t)(run0 - p.b_lo) * J0 * P1 + col;
#pragma unroll
          for (int a = 0; a < kYA; ++a) {
            if (a < J0) dst[(int64_t)a * P1] = yacc[u][a];
            yacc[u][a] = 0.f;
          }
        }
      }
    }
    if (run_end) run0 = b + 1;
    __syncthreads();  // Zs / u0t consumed
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

// ---------------------------------------------------------------------------
// k_spttmc4s: k_spttmc4t's arithmetic with the per-chunk phases on separate warp groups, so
// they overlap: warps 0-7 (leaf) build the plain fiber sums of chunk q + 1 into one of two T
// buffers while warps 8-11 (transpose) write chunk q's split K-major operands and one of them
// issues its tcgen05 MMAs; mbarriers hand the T buffers back and forth.  At a batch's end the
// transpose warps read Z out of TMEM into shared memory and the leaf warps run level 3 (Y in
// registers, as before) before the next batch.
// ---------------------------------------------------------------------------
constexpr int kSL = 256, kSX = 256, kSNT = kSL + kSX;  // leaf threads, transpose threads
constexpr int kCapS = 1024;                            // staged nonzeros per chunk buffer

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int CL>
__global__ void __launch_bounds__(kSNT, 1) k_spttmc4s(G4tArgs p) {
  extern __shared__ uint8_t sms_raw[];
  uint8_t* sms = sms_raw + ((1024u - (tc::smem_u32(sms_raw) & 1023u)) & 1023u);
  constexpr int kST = 3;  // bulk-copy stages (chunk data arrives two chunks ahead)
  __shared__ __align__(8) uint64_t full[kST], tpf[2], tpe[2], mma_done;
  __shared__ int st_e0[kST], st_ok[kST];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int JLP = 4 * CL, NB = 256 / JLP;
  constexpr int nslot = NB * kTKC;
  const int J0 = p.J0, J0P = p.J0P, J1 = p.J1;
  const int P1 = J1 * JLP;
  // layout: A_hi[2 tiles] A_lo[2 tiles] | B_hi B_lo | Tp[2] | Zs | Uls | u0t[3] | stage[3] | chunk bounds
  uint8_t* Ahi = sms;
  uint8_t* Alo = Ahi + 2 * kTA;
  uint8_t* Bhi = Alo + 2 * kTA;
  uint8_t* Blo = Bhi + kTB;
  float* Tp = reinterpret_cast<float*>(Blo + kTB);
  float* Zs = Tp + 2 * kTKC * kTpLd;
  float* Uls = Zs + ((NB * P1 + 3) & ~3);
  float* u0t = Uls + p.I_leaf * JLP;
  const int U0S = (NB * J0P + 3) & ~3;
  int* stg = reinterpret_cast<int*>(u0t + 3 * U0S);  // u0t[3]: batch b's rows in u0t[(b - b0) % 3]
  const int SB = 2 * p.SPC + 2 * kCapS;
  int* bnd = stg + kST * SB;  // nonzero offset of every chunk of this CTA (+ the end)

  const int b0 = p.b_lo + cta_first(blockIdx.x, p.nb, gridDim.x);
  const int b1 = p.b_lo + cta_first(blockIdx.x + 1, p.nb, gridDim.x);
  if (b0 >= b1) return;
  const int64_t ck0 = (int64_t)b0 * p.NCH, nck = (int64_t)(b1 - b0) * p.NCH;
  for (int64_t i = tid; i <= nck; i += kSNT) bnd[i] = __ldg(p.sp + (ck0 + i) * p.SPC);
  // chunks q + 2 .. q + 5 are prefetched into L2 ahead of their bulk copies into shared memory
  // (a chunk's work is ~1 us: two chunks of shared-memory lookahead do not cover HBM latency)
  auto prefetch = [&](int64_t q) {
    if (q >= nck) return;
    bulk_prefetch_l2(p.sp + (ck0 + q) * p.SPC, (uint32_t)(p.SPC * 4));
    bulk_prefetch_l2(p.tgt + (ck0 + q) * p.SPC, (uint32_t)(p.SPC * 4));
    const int E0r = bnd[q] & ~3, E1r = (bnd[q + 1] + 3) & ~3;
    if (E1r > E0r) {
      bulk_prefetch_l2(p.leaf + E0r, (uint32_t)(4 * (E1r - E0r)));
      bulk_prefetch_l2(p.val + E0r, (uint32_t)(4 * (E1r - E0r)));
    }
  };
  auto issue = [&](int64_t q, int E0, int E1) {
    const int buf = (int)(q % kST);
    int* sb = stg + buf * SB;
    const int E0r = E0 & ~3, E1r = (E1 + 3) & ~3;
    const int n = E1r - E0r;
    const bool ok = n <= kCapS;
    st_e0[buf] = E0r;
    st_ok[buf] = ok ? 1 : 0;
    tc::mbar_expect_tx(&full[buf], (uint32_t)(p.SPC * 8 + (ok ? 8 * n : 0)));
    bulk_g2s(sb, p.sp + (ck0 + q) * p.SPC, (uint32_t)(p.SPC * 4), &full[buf]);
    bulk_g2s(sb + p.SPC, p.tgt + (ck0 + q) * p.SPC, (uint32_t)(p.SPC * 4), &full[buf]);
    if (ok && n > 0) {
      bulk_g2s(sb + 2 * p.SPC, p.leaf + E0r, (uint32_t)(4 * n), &full[buf]);
      bulk_g2s(sb + 2 * p.SPC + kCapS, p.val + E0r, (uint32_t)(4 * n), &full[buf]);
    }
  };
  if (tid == 0) {
    for (int b = 0; b < kST; ++b) tc::mbar_init(&full[b], 1);
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tpf[b], kSL / 32);
      tc::mbar_init(&tpe[b], kSX / 32);
    }
    tc::mbar_init(&mma_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 8) {  // (k_spttmc4s: the first transpose warp)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tmem_slot)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int e = tid; e < p.I_leaf * JLP; e += kSNT) {
    const int r = e / JLP, j = e - r * JLP;
    Uls[e] = j < p.Jl ? __ldg(p.Ul + (int64_t)r * p.Jl + j) : 0.f;
  }
  for (int o = tid * 16; o < 4 * kTA + 2 * kTB; o += kSNT * 16) *reinterpret_cast<float4*>(sms + o) = make_float4(0.f, 0.f, 0.f, 0.f);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp < 8) {
    // ================= leaf group: T chunks, then level 3 at each batch's end
    if (tid == 0) {
      for (int64_t q = 0; q < kST && q < nck; ++q) issue(q, bnd[q], bnd[q + 1]);
      for (int64_t q = kST; q < kST + 4; ++q) prefetch(q);
    }
    // U_mid0 rows of batch b: loaded one batch ahead into u0t[(b - b0) % 3] (the transpose warps
    // read batch b's at its end, at most one batch behind)
    auto load_u0 = [&](int b) {
      if (b >= b1) return;
      const int4 bt = p.batch[b];
      float* u0b = u0t + ((b - b0) % 3) * U0S;
      for (int e = tid; e < NB * J0P; e += kSL) {
        const int v = e / J0P, a = e - v * J0P;
        u0b[e] = (v < bt.z && a < J0) ? __ldg(p.U0 + (int64_t)__ldg(p.node_mid0 + bt.y + v) * J0 + a) : 0.f;
      }
    };
    load_u0(b0);
    int64_t q = 0;
    for (int b = b0; b < b1; ++b) {
      const int4 bt = p.batch[b];
      load_u0(b + 1);
      for (int kc = 0; kc < p.NCH; ++kc, ++q) {
        const int tb = (int)(q & 1);
        const uint32_t use = (uint32_t)(q >> 1);
        const int sbuf = (int)(q % kST);
        tc::mbar_wait(&full[sbuf], (uint32_t)((q / kST) & 1));
        tc::mbar_wait(&tpe[tb], (use & 1) ^ 1);  // the transpose warps are done with T[tb]
        const int* sb = stg + sbuf * SB;
        const int E0r = st_e0[sbuf];
        const bool ok = st_ok[sbuf] != 0;
        float* T = Tp + tb * kTKC * kTpLd;
        for (int sl = tid; sl < ((p.dbg & 1) ? 0 : nslot); sl += kSL) {
          const int e0 = sb[sl], e1 = sb[sl + 1];
          const int tg = sb[p.SPC + sl];
          const int v = tg % NB, bl = tg / NB;
          float4 t[CL];
#pragma unroll
          for (int c = 0; c < CL; ++c) t[c] = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int e = e0; e < e1; ++e) {
            int l;
            float x;
            if (ok) {
              l = sb[2 * p.SPC + e - E0r];
              x = __int_as_float(sb[2 * p.SPC + kCapS + e - E0r]);
            } else {
              l = __ldg(p.leaf + e);
              x = __ldg(p.val + e);
            }
            const float4* r4 = reinterpret_cast<const float4*>(Uls + l * JLP);
#pragma unroll
            for (int c = 0; c < CL; ++c) {
              const float4 g = r4[c];
              t[c].x = fmaf(x, g.x, t[c].x);
              t[c].y = fmaf(x, g.y, t[c].y);
              t[c].z = fmaf(x, g.z, t[c].z);
              t[c].w = fmaf(x, g.w, t[c].w);
            }
          }
          float4* Tw = reinterpret_cast<float4*>(T + bl * kTpLd + v * JLP);
#pragma unroll
          for (int c = 0; c < CL; ++c) Tw[c] = t[c];
        }
        named_sync(1, kSL);  // T[tb] written; stage buffer tb free
        if (tid == 0 && q + kST < nck) {  // stage buffer sbuf is free: chunk q + 3 into it
          issue(q + kST, bnd[q + kST], bnd[q + kST + 1]);
          prefetch(q + kST + 4);
        }
        if (lane == 0) tc::mbar_arrive(&tpf[tb]);
      }
    }
  } else {
    // ================= transpose group: operands, MMAs, Z out of TMEM
    const int xt = tid - kSL, xw = xt >> 5;  // warp xw of the group: TMEM lane quarter xw & 3, Z tile xw >> 2
    const uint32_t sA = tc::smem_u32(Ahi), sAl = tc::smem_u32(Alo), sB = tc::smem_u32(Bhi), sBl = tc::smem_u32(Blo);
    const int k = lane;
    uint32_t o4[2][4];  // in-atom offsets of rows h + u at column k, h = 0 / 4
#pragma unroll
    for (int hh = 0; hh < 2; ++hh)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = 4 * hh + u;
        o4[hh][u] = (uint32_t)(r * 128 + ((((k >> 2) ^ r) << 4) | ((k & 3) << 2)));
      }
    uint32_t mphase = 0;
    bool pending = false;
    int64_t q = 0;
    constexpr int rows = NB * JLP;
    constexpr int kYC = 2, kYA = 24;  // Y columns xt + 256 u (J1 JLP <= 512), rows a < J0 <= 24
    float yacc[kYC][kYA];
#pragma unroll
    for (int u = 0; u < kYC; ++u)
#pragma unroll
      for (int a = 0; a < kYA; ++a) yacc[u][a] = 0.f;
    int run0 = b0;
    for (int b = b0; b < b1; ++b) {
      const int4 bt = p.batch[b];
      for (int kc = 0; kc < p.NCH; ++kc, ++q) {
        const int tb = (int)(q & 1);
        tc::mbar_wait(&tpf[tb], (uint32_t)((q >> 1) & 1));
        if (pending) {  // the previous chunk's MMAs have read A and B
          tc::mbar_wait(&mma_done, mphase & 1);
          ++mphase;
          pending = false;
        }
        const float* T = Tp + tb * kTKC * kTpLd;
        for (int r4 = xw; r4 < ((p.dbg & 2) ? 0 : rows / 4); r4 += kSX / 32) {
          const float4 v4 = *reinterpret_cast<const float4*>(T + k * kTpLd + 4 * r4);
          const int r0 = 4 * r4;
          const uint32_t base = (uint32_t)((r0 >> 7) * kTA + ((r0 & 127) >> 3) * 1024);
          const int hh = r4 & 1;
          t_split(Ahi, Alo, base + o4[hh][0], v4.x);
          t_split(Ahi, Alo, base + o4[hh][1], v4.y);
          t_split(Ahi, Alo, base + o4[hh][2], v4.z);
          t_split(Ahi, Alo, base + o4[hh][3], v4.w);
        }
        {
          const int bb = kc * kTKC + k;
          for (int r = xw; r < 32; r += kSX / 32) {
            const float u = (r < J1 && bb < p.I_mid1) ? __ldg(p.U1 + (int64_t)bb * J1 + r) : 0.f;
            t_split(Bhi, Blo, t_sw128(r, k), u);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&tpe[tb]);  // T[tb] may be refilled
        named_sync(2, kSX);                          // every operand write is done
        if (xt == 0 && !(p.dbg & 4)) {
          tc::tc_fence_after();
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            const uint32_t d = tmem + 32 * mt;
#pragma unroll
            for (int ks = 0; ks < kTKC / 8; ++ks) {
              const uint32_t o = (uint32_t)(ks * 32);
              const uint32_t ah = sA + mt * kTA + o, al = sAl + mt * kTA + o;
              tc::umma_tf32(d, tc::sw128_desc(ah), tc::sw128_desc(sB + o), kTIdesc, (kc > 0 || ks > 0) ? 1u : 0u);
              tc::umma_tf32(d, tc::sw128_desc(ah), tc::sw128_desc(sBl + o), kTIdesc, 1u);
              tc::umma_tf32(d, tc::sw128_desc(al), tc::sw128_desc(sB + o), kTIdesc, 1u);
            }
          }
          tc::umma_commit(&mma_done);
        }
        if (xt == 0 && (p.dbg & 4)) tc::mbar_arrive(&mma_done);
        pending = true;
      }
      // the batch's Z: TMEM row (v, c) of tile mt -> Zs[v][b' JLP + c]
      tc::mbar_wait(&mma_done, mphase & 1);
      ++mphase;
      pending = false;
      tc::tc_fence_after();
      {
        const int mt = xw >> 2, lq = xw & 3;
        float z[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * lq) << 16) + (uint32_t)(32 * mt), z);
        tc::tmem_wait_ld();
        const int r = mt * 128 + lq * 32 + lane;
        const int v = r / JLP, c = r - v * JLP;
        if (v < bt.z) {
#pragma unroll
          for (int bp = 0; bp < 32; ++bp)
            if (bp < J1) Zs[v * P1 + bp * JLP + c] = z[bp];
        }
      }
      tc::tc_fence_before();
      named_sync(2, kSX);  // Zs complete
      // ---- level 3: Y[a][col] += sum_v U_mid0[a_v][a] Z_v[col] (registers of the transpose warps)
      const float* u0b = u0t + ((b - b0) % 3) * U0S;
      const bool run_end = b + 1 == b1 || p.batch[b + 1].x != bt.x;
#pragma unroll
      for (int u = 0; u < kYC; ++u) {
        const int col = xt + kSX * u;
        if (col < P1) {
          for (int v = 0; v < ((p.dbg & 8) ? 0 : bt.z); ++v) {
            const float zz = Zs[v * P1 + col];
            const float4* u4 = reinterpret_cast<const float4*>(u0b + v * J0P);
#pragma unroll
            for (int a4 = 0; a4 < kYA / 4; ++a4) {
              if (4 * a4 < J0) {
                const float4 w = u4[a4];
                yacc[u][4 * a4] = fmaf(w.x, zz, yacc[u][4 * a4]);
                yacc[u][4 * a4 + 1] = fmaf(w.y, zz, yacc[u][4 * a4 + 1]);
                yacc[u][4 * a4 + 2] = fmaf(w.z, zz, yacc[u][4 * a4 + 2]);
                yacc[u][4 * a4 + 3] = fmaf(w.w, zz, yacc[u][4 * a4 + 3]);
              }
            }
          }
          if (run_end) {
            float* dst = p.part + (int64_t)(run0 - p.b_lo) * J0 * P1 + col;
#pragma unroll
            for (int a = 0; a < kYA; ++a) {
              if (a < J0) dst[(int64_t)a * P1] = yacc[u][a];
              yacc[u][a] = 0.f;
            }
          }
        }
      }
      if (run_end) run0 = b + 1;
      named_sync(2, kSX);  // Zs consumed before the next batch's Z
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

// ---- dense batch layout builder ----
__global__ void k_g4_node(const int32_t* __restrict__ slice_ptr, int64_t nslice, const int32_t* __restrict__ bfirst,
                          int64_t nnode, int NB, int NCH, int SPC, int32_t* __restrict__ node_base) {
  const int64_t nd = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (nd >= nnode) return;
  int64_t lo = 0, hi = nslice;  // slice s: slice_ptr[s] <= nd < slice_ptr[s + 1]
  while (hi - lo > 1) {
    const int64_t m = (lo + hi) / 2;
    if (slice_ptr[m] <= nd) lo = m;
    else hi = m;
  }
  const int vl = (int)(nd - slice_ptr[lo]);
  const int b = bfirst[lo] + vl / NB, v = vl % NB;
  node_base[nd] = (int32_t)((int64_t)b * NCH * SPC + v);
}

__global__ void k_g4_fiber(const int32_t* __restrict__ node_ptr, int64_t nnode, const int32_t* __restrict__ fib_ptr,
                           const int32_t* __restrict__ fib_mid1, int64_t nfib, const int32_t* __restrict__ node_base,
                           int NB, int SPC, int kch, int32_t* __restrict__ cnt, int32_t* __restrict__ fslot) {
  const int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f >= nfib) return;
  int64_t lo = 0, hi = nnode;
  while (hi - lo > 1) {
    const int64_t m = (lo + hi) / 2;
    if (node_ptr[m] <= f) lo = m;
    else hi = m;
  }
  const int b = fib_mid1[f];
  const int s = node_base[lo] + (b / kch) * SPC + (b % kch) * NB;
  cnt[s] = fib_ptr[f + 1] - fib_ptr[f];
  fslot[f] = s;
}

__global__ void k_g4_remap(int32_t* __restrict__ fslot, int64_t nfib, const int32_t* __restrict__ pos) {
  const int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f < nfib) fslot[f] = pos[fslot[f]];
}
static int bits_needed(uint64_t v) {
  int b = 1;
  while (b < 63 && (v >> b) != 0) ++b;
  return b;
}

// slots of each chunk sorted by nonzero count (descending; stable: padding slots last), so a
// warp's 32 consecutive slots have nearly equal loop trip counts
__global__ void k_g4_key(const int32_t* __restrict__ cnt, int64_t nslots, int SPC, uint32_t* __restrict__ key,
                         int32_t* __restrict__ id) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nslots) return;
  const uint32_t ch = (uint32_t)(t / SPC);
  key[t] = (ch << 10) | (uint32_t)(1023 - min(cnt[t], 1023));
  id[t] = (int32_t)t;
}
__global__ void k_g4_perm(const int32_t* __restrict__ sid, int64_t nslots, int SPC, const int32_t* __restrict__ cnt,
                          int32_t* __restrict__ cnt2, int32_t* __restrict__ tgt, int32_t* __restrict__ pos) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // sorted position
  if (q >= nslots) return;
  const int32_t s = sid[q];
  cnt2[q] = cnt[s];
  tgt[q] = (int32_t)(s % SPC);  // the slot's (b_local, v) index in its chunk
  pos[s] = (int32_t)q;
}

__global__ void k_g4_scatter(const int32_t* __restrict__ fib_ptr, int64_t nfib, const int32_t* __restrict__ fslot,
                             const int32_t* __restrict__ sp, const int32_t* __restrict__ leaf_id,
                             const float* __restrict__ val, int32_t* __restrict__ leaf2, float* __restrict__ val2) {
  const int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f >= nfib) return;
  const int e0 = fib_ptr[f], e1 = fib_ptr[f + 1];
  const int d = sp[fslot[f]];
  for (int e = e0; e < e1; ++e) {
    leaf2[d + e - e0] = leaf_id[e];
    val2[d + e - e0] = val[e];
  }
}

}  // namespace

// bytes of dynamic shared memory of k_spttmc4g
static size_t g4_smem(const Csf& c, int J0, int J1, int Jl, int NB, int SPC) {
  const int JLP = (int)round_up(Jl, 4), J1P = (int)round_up(J1, 4), J0P = (int)round_up(J0, 4);
  const int64_t P1 = (int64_t)J1 * JLP, P = (int64_t)J0 * P1;
  const int64_t tz = std::max<int64_t>((int64_t)kKCH * NB * JLP, NB * P1);
  const int64_t fl = c.I_leaf * JLP + c.I_mid1 * J1P + round_up(tz, 4) + round_up(P, 4) + (int64_t)NB * J0P;
  return (size_t)(fl + 2 * (2 * SPC + 2 * kCap)) * 4;
}

// bytes of dynamic shared memory of k_spttmc4t
static size_t g4t_smem(const Csf& c, int J0, int Jl, int NB, int SPC, bool bres) {
  const int JLP = (int)round_up(Jl, 4), J0P = (int)round_up(J0, 4);
  const int64_t fl = (int64_t)kTKC * kTpLd + c.I_leaf * JLP + round_up((int64_t)NB * J0P, 4);
  const size_t b = bres ? 1024 + (size_t)ceil_div(c.I_mid1, kTKC) * 2 * kTB : 0;
  return 1024 + 4 * kTA + 2 * kTB + (size_t)(fl + 2 * (2 * SPC + 2 * kCap)) * 4 + b;
}

// bytes of dynamic shared memory of k_spttmc4s
static size_t g4s_smem(const Csf& c, int J0, int J1, int Jl, int NB, int SPC, int maxck) {
  const int JLP = (int)round_up(Jl, 4), J0P = (int)round_up(J0, 4);
  const int64_t fl = 2 * (int64_t)kTKC * kTpLd + round_up((int64_t)NB * J1 * JLP, 4) + c.I_leaf * JLP +
                     3 * round_up((int64_t)NB * J0P, 4);
  return 1024 + 4 * kTA + 2 * kTB + (size_t)(fl + 3 * (2 * SPC + 2 * kCapS)) * 4 + (size_t)maxck * 4;
}

// The dense batch layout of ordering c for (NB nodes per batch, KCH mid1 indices per chunk),
// built on first use; false: too many slots for int32 offsets
static bool g4_layout(const Csf& c, int NB, int KCH, cudaStream_t st) {
  Csf::G4& g = *c.g4;
  if (g.nb_ == NB && g.kch == KCH) return true;
  const int NCH = (int)ceil_div(c.I_mid1, KCH);
  const int SPC = (int)round_up((int64_t)NB * KCH + 1, 4);
  std::vector<int32_t> sptr((size_t)c.I_root + 1);
  TK_CUDA(cudaMemcpyAsync(sptr.data(), c.slice_ptr.p, sptr.size() * 4, cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  std::vector<int4> batch;
  std::vector<int32_t> bfirst((size_t)c.I_root + 1);
  for (int64_t i = 0; i < c.I_root; ++i) {
    bfirst[i] = (int32_t)batch.size();
    for (int32_t n = sptr[i]; n < sptr[i + 1]; n += NB) batch.push_back(make_int4((int)i, n, std::min(NB, sptr[i + 1] - n), 0));
  }
  bfirst[c.I_root] = (int32_t)batch.size();
  const int64_t nbatch = (int64_t)batch.size();
  const int64_t nslots = nbatch * NCH * SPC;
  if (nslots + 8 >= (int64_t)1 << 31) return false;
  g.batch.alloc(std::max<int64_t>(1, nbatch));
  g.bfirst.alloc(bfirst.size());
  if (nbatch) TK_CUDA(cudaMemcpyAsync(g.batch.p, batch.data(), nbatch * sizeof(int4), cudaMemcpyHostToDevice, st));
  TK_CUDA(cudaMemcpyAsync(g.bfirst.p, bfirst.data(), bfirst.size() * 4, cudaMemcpyHostToDevice, st));
  DBuf<int32_t> node_base(std::max<int64_t>(1, c.nnode)), cnt(nslots + 8), fslot(std::max<int64_t>(1, c.nfib));
  g.sp.alloc(nslots + 8);
  TK_CUDA(cudaMemsetAsync(cnt.p, 0, (nslots + 8) * 4, st));
  if (c.nnode)
    TK_LAUNCH(k_g4_node, (unsigned)ceil_div(c.nnode, 256), 256, 0, st, c.slice_ptr.p, c.I_root, g.bfirst.p, c.nnode,
              NB, NCH, SPC, node_base.p);
  if (c.nfib)
    TK_LAUNCH(k_g4_fiber, (unsigned)ceil_div(c.nfib, 256), 256, 0, st, c.node_ptr.p, c.nnode, c.fib_ptr.p,
              c.fib_mid1.p, c.nfib, node_base.p, NB, SPC, KCH, cnt.p, fslot.p);
  // sort each chunk's slots by count (stable radix sort of (chunk, 1023 - count) keys)
  {
    DBuf<uint32_t> key(nslots), key2(nslots);
    DBuf<int32_t> id(nslots), id2(nslots), cnt2(nslots + 8), pos(nslots);
    g.tgt.alloc(nslots + 8);
    TK_CUDA(cudaMemsetAsync(g.tgt.p, 0, (nslots + 8) * 4, st));
    TK_LAUNCH(k_g4_key, (unsigned)ceil_div(nslots, 256), 256, 0, st, cnt.p, nslots, SPC, key.p, id.p);
    const int kbits = 10 + bits_needed((uint64_t)nbatch * NCH);
    size_t sb = 0;
    TK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sb, key.p, key2.p, id.p, id2.p, (int)nslots, 0, kbits, st));
    DBuf<uint8_t> stmp(sb);
    TK_CUDA(cub::DeviceRadixSort::SortPairs(stmp.p, sb, key.p, key2.p, id.p, id2.p, (int)nslots, 0, kbits, st));
    TK_CUDA(cudaMemsetAsync(cnt2.p, 0, (nslots + 8) * 4, st));
    TK_LAUNCH(k_g4_perm, (unsigned)ceil_div(nslots, 256), 256, 0, st, id2.p, nslots, SPC, cnt.p, cnt2.p, g.tgt.p, pos.p);
    // fslot: natural slot -> sorted position
    if (c.nfib) TK_LAUNCH(k_g4_remap, (unsigned)ceil_div(c.nfib, 256), 256, 0, st, fslot.p, c.nfib, pos.p);
    TK_CUDA(cudaMemcpyAsync(cnt.p, cnt2.p, (nslots + 8) * 4, cudaMemcpyDeviceToDevice, st));
  }
  size_t bytes = 0;
  TK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, g.sp.p, (int)(nslots + 8), st));
  DBuf<uint8_t> tmp(bytes);
  TK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.p, g.sp.p, (int)(nslots + 8), st));
  g.leaf.alloc(c.nnz + 8);
  g.val.alloc(c.nnz + 8);
  TK_CUDA(cudaMemsetAsync(g.leaf.p, 0, (c.nnz + 8) * 4, st));
  TK_CUDA(cudaMemsetAsync(g.val.p, 0, (c.nnz + 8) * 4, st));
  if (c.nfib)
    TK_LAUNCH(k_g4_scatter, (unsigned)ceil_div(c.nfib, 256), 256, 0, st, c.fib_ptr.p, c.nfib, fslot.p, g.sp.p,
              c.leaf_id.p, c.val.p, g.leaf.p, g.val.p);
  g.bfirst_h = bfirst;
  g.nbatch = nbatch;
  g.nb_ = NB;
  g.kch = KCH;
  return true;
}

// Run the GEMM-form SpTTMc (building the ordering's dense batch layout on first use); false =
// not applicable (the caller falls back to k_spttmc4w).  Default: the FMA kernel (k_spttmc4g);
// TUCKER_TTMC4=t selects the tcgen05 kernel (k_spttmc4t), =g the FMA kernel even where the
// density test would reject it, =w disables both (tests).
// True when spttmc4g would take the default FMA kernel on ordering c (the kernel that can keep Z)
bool spttmc4g_fma_default(const Csf& c, const int64_t* J) {
  const char* fe = std::getenv("TUCKER_TTMC4");
  const char fc = fe ? fe[0] : 0;  // 'g' forces the FMA kernel (tests); any other choice has no Z
  if ((fc != 0 && fc != 'g') || std::getenv("TUCKER_TTMC4_CS") || std::getenv("TUCKER_TTMC4_GMEM")) return false;
  if (c.order != 4) return false;
  const int J0 = (int)J[c.mid0], J1 = (int)J[c.mid1], Jl = (int)J[c.leaf];
  const int JLP = (int)round_up(Jl, 4), J1P = (int)round_up(J1, 4), CL = JLP / 4;
  if (CL > 8 || J0 > 256) return false;
  if (fc == 0 && (double)c.nnode * (double)round_up(c.I_mid1, 32) > 2.5 * (double)c.nfib) return false;
  const int NBg = kNT / CL;
  const int SPCg = (int)round_up((int64_t)NBg * kKCH + 1, 4);
  if (!(J1P <= 24 && g4_smem(c, J0, J1, Jl, NBg, SPCg) <= 220 * 1024)) return false;
  const int64_t nbatch_est = c.nnode / NBg + c.I_root;
  return (nbatch_est * ceil_div(c.I_mid1, kKCH) * SPCg + 8) < ((int64_t)1 << 31);
}

bool spttmc4g(const Csf& c, const float* const* U, const int64_t* J, Split out, bool transposed, int64_t s0,
              int64_t s1, int64_t sb, cudaStream_t st, int64_t lo, int64_t hi, float* zout) {
  const char* fe = std::getenv("TUCKER_TTMC4");
  const char fc = fe ? fe[0] : 0;
  if (fc == 'w' || c.order != 4) return false;
  const int J0 = (int)J[c.mid0], J1 = (int)J[c.mid1], Jl = (int)J[c.leaf];
  const int JLP = (int)round_up(Jl, 4), J1P = (int)round_up(J1, 4), CL = JLP / 4;
  if (CL > 8 || J0 > 256) return false;
  // density: slots (nodes x I_mid1) against fibers
  const double slots_est = (double)c.nnode * (double)round_up(c.I_mid1, 32);
  if (fc == 0 && slots_est > 2.5 * (double)c.nfib) return false;
  // tcgen05: N = 32 >= J1, rows NB JLP <= 256, Y columns J1 JLP <= 512 and J0 <= 32 in registers
  const int NBt = 256 / JLP;
  const int SPCt = (int)round_up((int64_t)NBt * kTKC + 1, 4);
  const bool bres = g4t_smem(c, J0, Jl, NBt, SPCt, true) <= 220 * 1024;
  const bool tc_ok = J1 <= 32 && J0 <= 32 && (int64_t)J1 * JLP <= 2 * kNT && g4t_smem(c, J0, Jl, NBt, SPCt, bres) <= 220 * 1024;
  const int NBg = kNT / CL;
  const int SPCg = (int)round_up((int64_t)NBg * kKCH + 1, 4);
  const bool g_ok = J1P <= 24 && g4_smem(c, J0, J1, Jl, NBg, SPCg) <= 220 * 1024;
  // default: the FMA kernel (measured at config 4: 0.51 ms per mode vs 0.65 ms for the tcgen05
  // kernel, whose per-chunk phases -- leaf, transpose, MMA issue -- are latency / barrier bound
  // with one 8-warp CTA per SM; tensor pipe 6 % busy)
  // (the transpose warps hold Y: J1 JLP <= 2 x 256 columns, J0 <= 24 rows; >= 3 chunks per batch keep
  // the leaf warps within one batch of them, so two U_mid0 buffers suffice)
  const int maxck_est = 1024;  // bound on chunks per CTA (4 KB of bounds), checked at launch
  const bool s_ok = J1 <= 32 && J0 <= 24 && (int64_t)J1 * JLP <= 2 * kSX && ceil_div(c.I_mid1, kTKC) >= 3 &&
                    g4s_smem(c, J0, J1, Jl, NBt, SPCt, maxck_est) <= 220 * 1024;
  const bool use_s = fc == 's' ? s_ok : false;
  const bool use_tc = use_s || (fc == 't' ? tc_ok : false);
  if (!use_tc && !g_ok) return false;
  if (zout && use_tc) fail(TUCKER_E_STATE, "spttmc4g: Z is kept by the FMA kernel only");
  if ((fc == 't' && !tc_ok) || (fc == 's' && !s_ok)) return false;
  const int NB = use_tc ? NBt : NBg, KCH = use_tc ? kTKC : kKCH, SPC = use_tc ? SPCt : SPCg;
  const int NCH = (int)ceil_div(c.I_mid1, KCH);
  if (!g4_layout(c, NB, KCH, st)) return false;
  Csf::G4& g = *c.g4;
  const int blo = g.bfirst_h[lo], bhi = g.bfirst_h[hi];
  const int nb = bhi - blo;
  const int64_t P = (int64_t)J0 * J1 * JLP;
  int nsm = 148, dev = 0;
  TK_CUDA(cudaGetDevice(&dev));
  TK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const int G = std::max(1, std::min(nb, nsm));
  if (nb > 0) {
    g.part.ensure((size_t)nb * P);
    if (use_tc) {
      G4tArgs a;
      a.batch = g.batch.p;
      a.node_mid0 = c.node_mid0.p;
      a.sp = g.sp.p;
      a.tgt = g.tgt.p;
      a.leaf = g.leaf.p;
      a.val = g.val.p;
      a.U0 = U[c.mid0];
      a.U1 = U[c.mid1];
      a.Ul = U[c.leaf];
      a.J0 = J0;
      a.J1 = J1;
      a.Jl = Jl;
      a.JLP = JLP;
      a.J0P = (int)round_up(J0, 4);
      a.CL = CL;
      a.NB = NB;
      a.NCH = NCH;
      a.SPC = SPC;
      a.I_leaf = (int)c.I_leaf;
      a.I_mid1 = (int)c.I_mid1;
      a.b_lo = blo;
      a.nb = nb;
      a.part = g.part.p;
      a.bres = bres ? 1 : 0;
      a.dbg = std::getenv("TUCKER_TTMC4_DBG") ? std::atoi(std::getenv("TUCKER_TTMC4_DBG")) : 0;
      if (use_s) {
        a.maxck = (int)(ceil_div(nb, G) * NCH + 8);
        if (a.maxck > maxck_est) fail(TUCKER_E_ARG, "spttmc4s: too many chunks per CTA");
        const size_t smem_s = g4s_smem(c, J0, J1, Jl, NB, SPC, a.maxck);
        switch (CL) {
#define TK_G4S(cl)                                                     \
  case cl:                                                             \
    smem_optin((const void*)k_spttmc4s<cl>, smem_s);                   \
    TK_LAUNCH(k_spttmc4s<cl>, (unsigned)G, kSNT, smem_s, st, a);       \
    break;
          TK_G4S(1) TK_G4S(2) TK_G4S(3) TK_G4S(4) TK_G4S(5) TK_G4S(6) TK_G4S(7) TK_G4S(8)
#undef TK_G4S
        }
      } else {
      const size_t smem = g4t_smem(c, J0, Jl, NB, SPC, bres);
      switch (CL) {
#define TK_G4T(cl)                                                     \
  case cl:                                                             \
    smem_optin((const void*)k_spttmc4t<cl>, smem);                     \
    TK_LAUNCH(k_spttmc4t<cl>, (unsigned)G, kNT, smem, st, a);          \
    break;
        TK_G4T(1) TK_G4T(2) TK_G4T(3) TK_G4T(4) TK_G4T(5) TK_G4T(6) TK_G4T(7) TK_G4T(8)
#undef TK_G4T
      }
      }
    } else {
      G4Args a;
      a.batch = g.batch.p;
      a.node_mid0 = c.node_mid0.p;
      a.sp = g.sp.p;
      a.tgt = g.tgt.p;
      a.leaf = g.leaf.p;
      a.val = g.val.p;
      a.U0 = U[c.mid0];
      a.U1 = U[c.mid1];
      a.Ul = U[c.leaf];
      a.J0 = J0;
      a.J1 = J1;
      a.Jl = Jl;
      a.JLP = JLP;
      a.J0P = (int)round_up(J0, 4);
      a.CL = CL;
      a.NB = NB;
      a.NCH = NCH;
      a.SPC = SPC;
      a.I_leaf = (int)c.I_leaf;
      a.I_mid1 = (int)c.I_mid1;
      a.b_lo = blo;
      a.nb = nb;
      a.part = g.part.p;
      a.zout = zout;
      const size_t smem = g4_smem(c, J0, J1, Jl, NB, SPC);
      bool launched = false;
#define TK_G4(j1p)                                                                  \
  if (!launched && J1P == j1p) {                                                    \
    smem_optin((const void*)k_spttmc4g<j1p>, smem);                                 \
    TK_LAUNCH(k_spttmc4g<j1p>, (unsigned)G, kNT, smem, st, a);                      \
    launched = true;                                                                \
  }
      TK_G4(4) TK_G4(8) TK_G4(12) TK_G4(16) TK_G4(20) TK_G4(24)
#undef TK_G4
    }
  }
  if (hi > lo) {
    const dim3 gr((unsigned)ceil_div(P, 256), (unsigned)(hi - lo));
    TK_LAUNCH(k_spttmc4g_reduce, gr, 256, 0, st, (const float*)g.part.p, (const int32_t*)g.bfirst.p, (int)lo, blo,
              std::max(nb, 1), G, J1, Jl, JLP, (int)P, s0, s1, sb, out.hi, out.lo, out.ld, (int)transposed);
  }
  return true;
}


// ---------------------------------------------------------------------------
// Sibling mode from the kept Z (HOOI partial-contraction reuse, order 4).
// Ordering (p; q; x; y): Z_v = X x_x U_x^T x_y U_y^T restricted to node v = (i_p, i_q).
// Mode p's row is Y_(p)[i_p] = sum_{i_q} U_q[i_q] (x) Z_v (level 3 above); the same Z gives
// mode q: Y_(q)[i_q] = sum_{i_p} U_p[i_p] (x) Z_v (Fig. 4 P:618-627 with Eq. 1 applied in
// another order), valid while U_x and U_y are unchanged -- in a Gauss-Seidel sweep exactly
// when q = p + 1.  Thread = one Z column and 16 U_p columns; the nodes of i_q in ascending
// i_p, one fixed-order sum per output (deterministic).  kSibJ: U_p columns per thread (one
// tile covers J_p <= 24, so Z is read once; larger J_p in tiles of 16).
// ---------------------------------------------------------------------------
constexpr int kSibT = 64, kSibN = 32, kSibU = 16;
template <int kSibJ>
__global__ void __launch_bounds__(kSibT) k_spttmc4_sib(const float* __restrict__ Z, const int32_t* __restrict__ sib_ptr,
                                                      const int32_t* __restrict__ sib_node,
                                                      const int32_t* __restrict__ node_root,
                                                      const float* __restrict__ Ur, int Jr, int J1, int Jl, int JLP,
                                                      int64_t sr, int64_t s1, int64_t sb, float* __restrict__ Yhi,
                                                      float* __restrict__ Ylo, int64_t ldY, int transposed) {
  __shared__ __align__(16) float us[kSibN][kSibJ];
  __shared__ int nd[kSibN];
  const int P1 = J1 * JLP;
  const int col = blockIdx.x * kSibT + threadIdx.x;
  const int a = blockIdx.y;
  const int jr0 = blockIdx.z * kSibJ;
  const bool live = col < P1;
  float y[kSibJ];
#pragma unroll
  for (int t = 0; t < kSibJ; ++t) y[t] = 0.f;
  const int k0 = sib_ptr[a], k1 = sib_ptr[a + 1];
  for (int kb = k0; kb < k1; kb += kSibN) {
    const int n = min(kSibN, k1 - kb);
    __syncthreads();
    if (threadIdx.x < n) nd[threadIdx.x] = sib_node[kb + threadIdx.x];
    for (int e = threadIdx.x; e < n * kSibJ; e += kSibT) {
      const int k = e / kSibJ, t = e - k * kSibJ;
      const int v = sib_node[kb + k];
      us[k][t] = jr0 + t < Jr ? __ldg(Ur + (int64_t)node_root[v] * Jr + jr0 + t) : 0.f;
    }
    __syncthreads();
    if (live) {
      int k = 0;
      for (; k + kSibU <= n; k += kSibU) {
        float z[kSibU];
#pragma unroll
        for (int u = 0; u < kSibU; ++u) z[u] = __ldg(Z + (int64_t)nd[k + u] * P1 + col);
#pragma unroll
        for (int u = 0; u < kSibU; ++u)
#pragma unroll
          for (int t4 = 0; t4 < kSibJ / 4; ++t4) {
            const float4 g = *reinterpret_cast<const float4*>(&us[k + u][4 * t4]);
            y[4 * t4] = fmaf(g.x, z[u], y[4 * t4]);
            y[4 * t4 + 1] = fmaf(g.y, z[u], y[4 * t4 + 1]);
            y[4 * t4 + 2] = fmaf(g.z, z[u], y[4 * t4 + 2]);
            y[4 * t4 + 3] = fmaf(g.w, z[u], y[4 * t4 + 3]);
          }
      }
      for (; k < n; ++k) {
        const float z = __ldg(Z + (int64_t)nd[k] * P1 + col);
#pragma unroll
        for (int t = 0; t < kSibJ; ++t) y[t] = fmaf(us[k][t], z, y[t]);
      }
    }
  }
  if (!live) return;
  const int r = col / JLP, c = col - r * JLP;
  if (c >= Jl) return;
#pragma unroll
  for (int t = 0; t < kSibJ; ++t) {
    if (jr0 + t >= Jr) break;
    const int64_t ycol = (jr0 + t) * sr + r * s1 + c * sb;
    const int64_t off = transposed ? ycol * ldY + a : (int64_t)a * ldY + ycol;
    const float h = tf32_rna_g4(y[t]);
    Yhi[off] = h;
    Ylo[off] = tf32_rna_g4(y[t] - h);
  }
}

__global__ void k_sib_node_root(const int32_t* __restrict__ slice_ptr, int64_t nslice, int64_t nnode,
                                int32_t* __restrict__ node_root, int32_t* __restrict__ id) {
  const int64_t nd = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (nd >= nnode) return;
  int64_t lo = 0, hi = nslice;
  while (hi - lo > 1) {
    const int64_t m = (lo + hi) / 2;
    if (slice_ptr[m] <= nd) lo = m;
    else hi = m;
  }
  node_root[nd] = (int32_t)lo;
  id[nd] = (int32_t)nd;
}
__global__ void k_sib_ptr(const int32_t* __restrict__ key, int64_t nnode, int64_t I, int32_t* __restrict__ ptr) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a > I) return;
  int64_t lo = 0, hi = nnode;  // first position with key >= a
  while (lo < hi) {
    const int64_t m = (lo + hi) / 2;
    if (key[m] < a) lo = m + 1;
    else hi = m;
  }
  ptr[a] = (int32_t)lo;
}

void spttmc4_sibling(const Csf& c, const float* Z, const float* Uroot, const int64_t* J, Split out, bool transposed,
                     int64_t sr, int64_t s1, int64_t sb, cudaStream_t st) {
  Csf::G4& g = *c.g4;
  if (!g.sib_built) {  // nodes grouped by mid0 (stable: ascending root inside a group)
    const int64_t nn = std::max<int64_t>(1, c.nnode);
    g.node_root.alloc(nn);
    g.sib_node.alloc(nn);
    g.sib_ptr.alloc(c.I_mid0 + 1);
    DBuf<int32_t> id(nn), key2(nn);
    if (c.nnode)
      TK_LAUNCH(k_sib_node_root, (unsigned)ceil_div(c.nnode, 256), 256, 0, st, c.slice_ptr.p, c.I_root, c.nnode,
                g.node_root.p, id.p);
    size_t sbytes = 0;
    TK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sbytes, c.node_mid0.p, key2.p, id.p, g.sib_node.p, (int)c.nnode, 0,
                                            bits_needed((uint64_t)c.I_mid0), st));
    DBuf<uint8_t> stmp(sbytes);
    TK_CUDA(cub::DeviceRadixSort::SortPairs(stmp.p, sbytes, c.node_mid0.p, key2.p, id.p, g.sib_node.p, (int)c.nnode, 0,
                                            bits_needed((uint64_t)c.I_mid0), st));
    TK_LAUNCH(k_sib_ptr, (unsigned)ceil_div(c.I_mid0 + 1, 256), 256, 0, st, (const int32_t*)key2.p, c.nnode, c.I_mid0,
              g.sib_ptr.p);
    TK_CUDA(cudaStreamSynchronize(st));  // the temporaries go out of scope
    g.sib_built = true;
  }
  const int Jr = (int)J[c.root], J1 = (int)J[c.mid1], Jl = (int)J[c.leaf];
  const int JLP = (int)round_up(Jl, 4);
  const int JT = Jr <= 8 ? 8 : (Jr <= 16 ? 16 : (Jr <= 24 ? 24 : 16));
  const dim3 gr((unsigned)ceil_div((int64_t)J1 * JLP, kSibT), (unsigned)c.I_mid0, (unsigned)ceil_div(Jr, JT));
#define TK_SIB(jt)                                                                                                   \
  if (JT == jt)                                                                                                      \
    TK_LAUNCH(k_spttmc4_sib<jt>, gr, kSibT, 0, st, Z, (const int32_t*)g.sib_ptr.p, (const int32_t*)g.sib_node.p,     \
              (const int32_t*)g.node_root.p, Uroot, Jr, J1, Jl, JLP, sr, s1, sb, out.hi, out.lo, out.ld,            \
              (int)transposed);
  TK_SIB(8) TK_SIB(16) TK_SIB(24)
#undef TK_SIB
}

}  // namespace tk
