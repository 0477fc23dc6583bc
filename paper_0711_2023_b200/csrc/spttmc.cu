// spttmc.cu -- sparse tensor-times-matrix kernels.
//
// HOOI (Fig. 4): Y_(n) = (X x_{m != n} U_m^T)_(n).  Per slice i of
// mode n (PAPER Appendix: row i of Y_(1) is B' * X1_slice * C):
//   order 3:  Y_i[a, b] = sum_{fibers f of slice i} U_mid[mid(f), a] * t_f[b],
//             t_f[b]    = sum_{x in f} x * U_leaf[leaf(x), b]           (Eq. 1)
//   order 4:  Y_i[a0, a1, b] = sum_{nodes v of i} U_mid0[mid0(v), a0] * Z_v[a1, b],
//             Z_v[a1, b] = sum_{fibers f of v} U_mid1[mid1(f), a1] * t_f[b]
// One CTA per slice; the fiber (leaf) stage gathers U_leaf rows with
// coalesced warp loads, the Kronecker stage is a register-tiled outer-product
// accumulation; no global atomics.  The output row is written once, split
// into (tf32 hi, tf32 lo) pairs for the 3xTF32 Gram.
//
// MP (Fig. 7/8, Appendix): W = (X x_m U_m^T)_(n), whose column
// block for the slice s fixing the modes not in {n, m} is X_s U_m.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <array>
#include <vector>

#include <cooperative_groups.h>

#include "internal.cuh"
#include "tc_ptx.cuh"

namespace cg = cooperative_groups;

namespace tk {

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void split_store(float* hi, float* lo, int64_t off, float y) {
  float h = tf32_rna(y);
  hi[off] = h;
  lo[off] = tf32_rna(y - h);
}

namespace {

constexpr int kFC = 32;  // fibers per chunk

// Leaf stage with the chunk's fiber metadata (fptr: nf + 1 nonzero offsets,
// fmid: mid indices) already in shared memory and, when the chunk's
// nonzeros fit (sl != nullptr), their leaf ids / values staged too: per
// fiber the only global hop left is the U row gathers.  Lane l gathers the
// VW-float vector at columns VW*l (+ 32 VW per pass) of each U_leaf row (one
// 64/128-bit load per nonzero and pass), UN nonzeros in flight at a time.
constexpr int kNS = 512;  // staged nonzeros per chunk
template <int VW>
struct FVec;
template <>
struct FVec<1> {
  using T = float;
  static __device__ __forceinline__ void fma(float x, T g, float* t) { t[0] = fmaf(x, g, t[0]); }
};
template <>
struct FVec<2> {
  using T = float2;
  static __device__ __forceinline__ void fma(float x, T g, float* t) {
    t[0] = fmaf(x, g.x, t[0]);
    t[1] = fmaf(x, g.y, t[1]);
  }
};
template <>
struct FVec<4> {
  using T = float4;
  static __device__ __forceinline__ void fma(float x, T g, float* t) {
    t[0] = fmaf(x, g.x, t[0]);
    t[1] = fmaf(x, g.y, t[1]);
    t[2] = fmaf(x, g.z, t[2]);
    t[3] = fmaf(x, g.w, t[3]);
  }
};

template <int VW, int QV, int UN>
__device__ __forceinline__ void gather_rows(const int* l, const float* x, int n,
                                            const float* __restrict__ Uleaf, int ldl, int Jl, int lane,
                                            float (&t)[QV][VW]) {
  using V = typename FVec<VW>::T;
  V g[UN][QV];
#pragma unroll
  for (int u = 0; u < UN; ++u) {
    const V* r = reinterpret_cast<const V*>(Uleaf + (int64_t)l[u] * ldl);
#pragma unroll
    for (int q = 0; q < QV; ++q) {
      const int v = lane + 32 * q;
      if (u < n && v * VW < Jl) g[u][q] = __ldg(r + v);
      else g[u][q] = V{};
    }
  }
#pragma unroll
  for (int u = 0; u < UN; ++u)
#pragma unroll
    for (int q = 0; q < QV; ++q) FVec<VW>::fma(x[u], g[u][q], t[q]);
}

template <int JLP, int JMP, int VW>
__device__ __forceinline__ void leaf_stage_s(int nf, const int* fptr, const int* fmid, const int* sl,
                                             const float* sv, const int32_t* __restrict__ leaf_id,
                                             const float* __restrict__ val,
                                             const float* __restrict__ Umid, int Jm,
                                             const float* __restrict__ Uleaf, int Jl, float* T,
                                             float* M) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  constexpr int QV = (JLP + 32 * VW - 1) / (32 * VW);
  constexpr int QM = (JMP + 31) / 32;
  constexpr int UN = 4;
  const int E0 = fptr[0];
  for (int fl = warp; fl < nf; fl += nwarps) {
    const int e0 = fptr[fl], e1 = fptr[fl + 1];
    const float* mr = Umid + (int64_t)fmid[fl] * Jm;
    float mv[QM];
#pragma unroll
    for (int q = 0; q < QM; ++q) {
      const int j = lane + 32 * q;
      mv[q] = (j < Jm) ? __ldg(mr + j) : 0.f;
    }
    float t[QV][VW];
#pragma unroll
    for (int q = 0; q < QV; ++q)
#pragma unroll
      for (int k = 0; k < VW; ++k) t[q][k] = 0.f;
    int l[UN];
    float x[UN];
    if (sl) {
      for (int e = e0; e < e1; e += UN) {
        const int n = min(UN, e1 - e);
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          l[u] = u < n ? sl[e + u - E0] : 0;
          x[u] = u < n ? sv[e + u - E0] : 0.f;
        }
        gather_rows<VW, QV, UN>(l, x, n, Uleaf, Jl, Jl, lane, t);
      }
    } else {
      for (int e = e0; e < e1; e += UN) {
        const int n = min(UN, e1 - e);
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          l[u] = u < n ? __ldg(leaf_id + e + u) : 0;
          x[u] = u < n ? __ldg(val + e + u) : 0.f;
        }
        gather_rows<VW, QV, UN>(l, x, n, Uleaf, Jl, Jl, lane, t);
      }
    }
#pragma unroll
    for (int q = 0; q < QV; ++q)
#pragma unroll
      for (int k = 0; k < VW; ++k) {
        const int j = (lane + 32 * q) * VW + k;
        if (j < JLP) T[fl * JLP + j] = t[q][k];
      }
#pragma unroll
    for (int q = 0; q < QM; ++q) {
      const int j = lane + 32 * q;
      if (j < JMP) M[fl * JMP + j] = mv[q];
    }
  }
}

// Kronecker stage over one chunk: acc[r][c] += M[fl][a(r)] * T[fl][b(c)].
// Thread (tx, ty) owns rows a(r) = ty*RA + r (contiguous: RA/4 broadcast
// 128-bit loads) and columns b(c) = (c/V)*16V + tx*V + c%V with V = min(RB, 4)
// (each vector load of a half-warp is one contiguous 16V-float run: no bank
// conflicts).  Per fiber a warp issues RA/4 + RB/V loads for RA*RB FFMAs.
template <int RB>
struct KronV {
  static constexpr int V = RB < 4 ? RB : 4;
};
template <int RA, int RB>
__device__ __forceinline__ int kron_col(int tx, int c) {
  constexpr int V = KronV<RB>::V;
  return (c / V) * 16 * V + tx * V + (c % V);
}
template <int RA, int RB>
__device__ __forceinline__ void kron_stage(int nf, const float* T, const float* M,
                                           float (&acc)[RA][RB]) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  constexpr int JLP = 16 * RB, JMP = 16 * RA;
  constexpr int V = KronV<RB>::V;
#pragma unroll 2
  for (int fl = 0; fl < nf; ++fl) {
    float a[RA], b[RB];
    const float* mr = M + fl * JMP + ty * RA;
    if constexpr (RA % 4 == 0) {
#pragma unroll
      for (int r = 0; r < RA; r += 4) {
        const float4 v = *reinterpret_cast<const float4*>(mr + r);
        a[r] = v.x; a[r + 1] = v.y; a[r + 2] = v.z; a[r + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int r = 0; r < RA; ++r) a[r] = mr[r];
    }
    const float* tr = T + fl * JLP + tx * V;
#pragma unroll
    for (int q = 0; q < RB / V; ++q) {
      if constexpr (V == 4) {
        const float4 v = *reinterpret_cast<const float4*>(tr + q * 16 * V);
        b[4 * q] = v.x; b[4 * q + 1] = v.y; b[4 * q + 2] = v.z; b[4 * q + 3] = v.w;
      } else if constexpr (V == 2) {
        const float2 v = *reinterpret_cast<const float2*>(tr + q * 16 * V);
        b[2 * q] = v.x; b[2 * q + 1] = v.y;
      } else {
        b[q] = tr[q * 16];
      }
    }
#pragma unroll
    for (int r = 0; r < RA; ++r)
#pragma unroll
      for (int c = 0; c < RB; ++c) acc[r][c] += a[r] * b[c];
  }
}

// Small cores (16 RA x 16 RB <= 512 outputs per slice): the 16 x 16 thread grid above leaves each
// thread 1-2 accumulators, i.e. ~3 shared loads and loop overhead per 1-2 FMAs in all 8 warps for every
// fiber (ncu at config 3 mode 1, 25 x 10 outputs: issue 83 %, FMA 36 %).  Here a chunk is 128 fibers,
// each warp runs the Kronecker update of 16 of them, lane = a BR x 4 block of the tile (two vector
// loads per 4 BR FMAs), and the 8 per-warp partial tiles are summed in warp order at the end
// (deterministic).
template <int RA, int RB>
struct KronSmall {
  static constexpr int JLP = 16 * RB, JMP = 16 * RA;
  static constexpr int CB = JLP / 4;        // 4-column blocks per row
  static constexpr int RBK = 32 / CB;       // row blocks
  static constexpr bool on = RA * RB <= 2;
  static constexpr int BR = on ? JMP / RBK : 1;  // rows per lane: 2 or 4
};
constexpr int kFCS = 128;  // fibers per chunk on the small-core path
template <int RA, int RB>
__device__ __forceinline__ void kron_small(int nf, const float* T, const float* M,
                                           float (&acc)[KronSmall<RA, RB>::BR][4]) {
  using K = KronSmall<RA, RB>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cb = lane % K::CB, rb = lane / K::CB;
  const int fl1 = min(nf, (warp + 1) * (kFCS / 8));
  for (int fl = warp * (kFCS / 8); fl < fl1; ++fl) {
    const float4 b = *reinterpret_cast<const float4*>(T + fl * K::JLP + 4 * cb);
    float a[K::BR];
    const float* mr = M + fl * K::JMP + rb * K::BR;
    if constexpr (K::BR == 4) {
      const float4 v = *reinterpret_cast<const float4*>(mr);
      a[0] = v.x; a[1] = v.y; a[2] = v.z; a[3] = v.w;
    } else {
      const float2 v = *reinterpret_cast<const float2*>(mr);
      a[0] = v.x; a[1] = v.y;
    }
#pragma unroll
    for (int r = 0; r < K::BR; ++r) {
      acc[r][0] += a[r] * b.x;
      acc[r][1] += a[r] * b.y;
      acc[r][2] += a[r] * b.z;
      acc[r][3] += a[r] * b.w;
    }
  }
}

// Small-core leaf stage, one LANE per fiber (the warp-per-fiber stage above keeps 5 of 32 lanes busy at
// J_leaf = 10 and spends ~60 instructions per fiber): t_f in registers, the U_leaf rows read as VW-float
// vectors (L1 / L2 hits: the table is I x J_leaf floats), then one padded row of T.
template <int JLP, int VW>
__device__ __forceinline__ void leaf_lane(int t, const int* fptr, const int* sl, const float* sv, int E0,
                                          const int32_t* __restrict__ leaf_id, const float* __restrict__ val,
                                          const float* __restrict__ Uleaf, int Jl, float* T) {
  using V = typename FVec<VW>::T;
  constexpr int NV = JLP / VW;
  float tt[JLP];
#pragma unroll
  for (int j = 0; j < JLP; ++j) tt[j] = 0.f;
  const int e0 = fptr[t], e1 = fptr[t + 1];
  for (int e = e0; e < e1; ++e) {
    int l;
    float x;
    if (sl) {
      l = sl[e - E0];
      x = sv[e - E0];
    } else {
      l = __ldg(leaf_id + e);
      x = __ldg(val + e);
    }
    const V* r = reinterpret_cast<const V*>(Uleaf + (int64_t)l * Jl);
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (v * VW < Jl) FVec<VW>::fma(x, __ldg(r + v), tt + v * VW);
  }
  float4* Tw = reinterpret_cast<float4*>(T + t * JLP);
#pragma unroll
  for (int q = 0; q < JLP / 4; ++q) Tw[q] = make_float4(tt[4 * q], tt[4 * q + 1], tt[4 * q + 2], tt[4 * q + 3]);
}
// the chunk's U_mid rows (zero padded to JMP <= 32), a warp per row, by the upper four warps
template <int JMP>
__device__ __forceinline__ void mid_rows(int nf, const int* fmid, const float* __restrict__ Umid, int Jm, float* M) {
  const int w = (threadIdx.x >> 5) - 4, lane = threadIdx.x & 31;
  for (int fl = w; fl < nf; fl += 4) {
    const float* mr = Umid + (int64_t)fmid[fl] * Jm;
    if (lane < JMP) M[fl * JMP + lane] = lane < Jm ? __ldg(mr + lane) : 0.f;
  }
}

struct Ttmc3Args {
  const int32_t *slice_ptr, *fib_ptr, *fib_mid, *leaf_id;
  const int32_t* unit;  // work units (slice, f0, f1, slot) or null: one CTA per slice
  int slice0;           // first slice of this launch (rank shard) when unit == null
  float* part;          // partial tiles of split slices (Jm * Jl floats per slot)
  const float* val;
  const float *Umid, *Uleaf;
  int Jm, Jl;
  float *Yhi, *Ylo;
  int64_t ldY;
  int transposed;
  int64_t sa, sb;  // Kolda strides of (mid index a, leaf index b) in the output column
  // k_spttmc3_tc column windows (J_mid or J_leaf > 128): Umid / Uleaf point at column a0 / b0 of
  // factors with row strides ldm / ldl; Jm / Jl are the window widths
  int ldm, ldl, a0, b0;
};

template <int RA, int RB, int VW>
__global__ void __launch_bounds__(256) k_spttmc3(Ttmc3Args p) {
  constexpr int JLP = 16 * RB, JMP = 16 * RA;
  constexpr int FC = KronSmall<RA, RB>::on ? kFCS : kFC;  // fibers per chunk
  __shared__ __align__(16) float T[FC * JLP];
  __shared__ __align__(16) float M[FC * JMP];
  int i, f0, f1, slot = -1;
  if (p.unit) {
    const int4 u = reinterpret_cast<const int4*>(p.unit)[blockIdx.x];
    i = u.x;
    f0 = u.y;
    f1 = u.z;
    slot = u.w;
  } else {
    i = p.slice0 + blockIdx.x;
    f0 = p.slice_ptr[i];
    f1 = p.slice_ptr[i + 1];
  }
  float acc[RA][RB];
#pragma unroll
  for (int r = 0; r < RA; ++r)
#pragma unroll
    for (int c = 0; c < RB; ++c) acc[r][c] = 0.f;
  using KS = KronSmall<RA, RB>;
  float acc2[KS::BR][4];  // small cores: this warp's partial BR x 4 block (kron_small)
#pragma unroll
  for (int r = 0; r < KS::BR; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc2[r][c] = 0.f;
  __shared__ int fptr[FC + 1], fmid[FC];
  __shared__ int sl[kNS];
  __shared__ float sv[kNS];
  // chunk metadata prefetched into registers one chunk ahead
  int nx_ptr = 0, nx_mid = 0;
  if (f0 < f1 && threadIdx.x <= min(FC, f1 - f0)) {
    nx_ptr = __ldg(p.fib_ptr + f0 + threadIdx.x);
    if (threadIdx.x < min(FC, f1 - f0)) nx_mid = __ldg(p.fib_mid + f0 + threadIdx.x);
  }
  for (int fc = f0; fc < f1; fc += FC) {
    const int nf = min(FC, f1 - fc);
    if (threadIdx.x <= nf) fptr[threadIdx.x] = nx_ptr;
    if (threadIdx.x < nf) fmid[threadIdx.x] = nx_mid;
    __syncthreads();
    const int E0 = fptr[0], E1 = fptr[nf];
    const bool staged = E1 - E0 <= kNS;
    if (staged)
      for (int e = E0 + (int)threadIdx.x; e < E1; e += blockDim.x) {
        sl[e - E0] = __ldg(p.leaf_id + e);
        sv[e - E0] = __ldg(p.val + e);
      }
    // next chunk's metadata: in flight during this chunk's stages
    const int fn = fc + FC;
    if (fn < f1) {
      const int nfn = min(FC, f1 - fn);
      if (threadIdx.x <= nfn) nx_ptr = __ldg(p.fib_ptr + fn + threadIdx.x);
      if (threadIdx.x < nfn) nx_mid = __ldg(p.fib_mid + fn + threadIdx.x);
    }
    __syncthreads();
    if constexpr (KS::on) {
      // lower four warps: one lane per fiber (t_f); upper four: the fibers' U_mid rows
      if (threadIdx.x < kFCS) {
        if ((int)threadIdx.x < nf)
          leaf_lane<JLP, VW>(threadIdx.x, fptr, staged ? sl : nullptr, sv, E0, p.leaf_id, p.val, p.Uleaf, p.Jl, T);
      } else {
        mid_rows<JMP>(nf, fmid, p.Umid, p.Jm, M);
      }
      __syncthreads();
      kron_small<RA, RB>(nf, T, M, acc2);
    } else {
      leaf_stage_s<JLP, JMP, VW>(nf, fptr, fmid, staged ? sl : nullptr, sv, p.leaf_id, p.val, p.Umid, p.Jm,
                                 p.Uleaf, p.Jl, T, M);
      __syncthreads();
      kron_stage<RA, RB>(nf, T, M, acc);
    }
    __syncthreads();
  }
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  if constexpr (KS::on) {  // the 8 warps' partial tiles, summed in warp order
    __shared__ __align__(16) float red[8][JMP * JLP];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cb = lane % KS::CB, rb = lane / KS::CB;
#pragma unroll
    for (int r = 0; r < KS::BR; ++r)
      *reinterpret_cast<float4*>(&red[warp][(rb * KS::BR + r) * JLP + 4 * cb]) =
          make_float4(acc2[r][0], acc2[r][1], acc2[r][2], acc2[r][3]);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RA; ++r)
#pragma unroll
      for (int c = 0; c < RB; ++c) {
        const int e = (ty * RA + r) * JLP + kron_col<RA, RB>(tx, c);
        float v = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) v += red[w][e];
        acc[r][c] = v;
      }
  }
#pragma unroll
  for (int r = 0; r < RA; ++r)
#pragma unroll
    for (int c = 0; c < RB; ++c) {
      const int a = ty * RA + r, b = kron_col<RA, RB>(tx, c);
      if (slot >= 0) {
        if (a < p.Jm && b < p.Jl) p.part[(int64_t)slot * p.Jm * p.Jl + a * p.Jl + b] = acc[r][c];
      } else if (a < p.Jm && b < p.Jl) {
        const int64_t col = a * p.sa + b * p.sb;
        const int64_t off = p.transposed ? col * p.ldY + i : (int64_t)i * p.ldY + col;
        split_store(p.Yhi, p.Ylo, off, acc[r][c]);
      }
    }
}

// ---------------------------------------------------------------------------
// Tensor-core Kronecker stage (order 3, J_mid, J_leaf <= 128).  Per chunk of
// KC = 32 fibers the Kronecker update Y_i += M_c^T T_c (M_c: KC x J_mid rows
// of U_mid, T_c: KC x J_leaf fiber sums t_f, Eq. 1) is a K = 32 contraction,
// run as 3xTF32 tcgen05 MMAs (hi.hi + hi.lo + lo.hi, fp32 accumulation in
// TMEM, D = 128 x N with row a = mid index, column b = leaf index).  Both
// operands are K-major with the 128-byte swizzle (the layout the Gram kernel
// uses): one operand row = one mid/leaf index, its 32 fibers = one 128-byte
// swizzle row, so the leaf stage stores fiber k's values into column k.  The
// TMEM accumulator is drained into fp32 registers every kTcGroup chunks and
// restarted (measured: accumulating a whole heavy slice in TMEM left Y with
// 3-5e-5 relative error at config 5 mode 3, against ~5e-7 for the SIMT kernel --
// the tensor core's accumulation is not an IEEE fp32 sum).  One
// operand buffer (so 3-4 CTAs fit per SM and the latency-bound gathers have
// warps to hide behind): the chunk's metadata staging overlaps the previous
// chunk's MMAs, and the operand stores wait for their commit.
// (MN-major tf32 operands would avoid the transposed stores, but produced
// zeros in tools/umma_mn_test.cu; K-major is the verified layout.)
// ---------------------------------------------------------------------------
constexpr int KC = 32;                // fibers (K) per chunk = one 128-byte swizzle row
constexpr int kTcGroup = 4;           // chunks accumulated in TMEM between drains into registers
constexpr int TC_A_BYTES = 128 * 128; // A: 128 rows (M) x 128 B

template <int NA>  // B: 32 NA rows (N = 32 NA)
struct TcTile {
  static constexpr int B_BYTES = 32 * NA * 128;
  static constexpr int BUF = 2 * TC_A_BYTES + 2 * B_BYTES;  // A_hi, A_lo, B_hi, B_lo
  static constexpr int SMEM = BUF + KC * 32 * NA * 4 + 1024;  // operands + plain t rows + alignment slack
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) |  // F32 <- TF32 x TF32, K-major
                                    ((uint32_t)(32 * NA) >> 3 << 17) | ((uint32_t)(128 >> 4) << 24);
  static constexpr int TMEM_COLS = NA <= 1 ? 32 : (NA <= 2 ? 64 : 128);
};

// byte offset of element (row, k) in a K-major SW128 tile (K = 32 per row)
__device__ __forceinline__ uint32_t k_sw128(int row, int k) {
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((((k >> 2) ^ (row & 7)) << 4) | ((k & 3) << 2)));
}

__device__ __forceinline__ void st_split1(uint8_t* hi, uint8_t* lo, uint32_t off, float v) {
  const float h = tf32_rna(v);
  *reinterpret_cast<float*>(hi + off) = h;
  *reinterpret_cast<float*>(lo + off) = tf32_rna(v - h);
}

template <int NA, int VW>
__global__ void __launch_bounds__(256) k_spttmc3_tc(Ttmc3Args p) {
  using Tile = TcTile<NA>;
  constexpr int QV = (32 * NA + 32 * VW - 1) / (32 * VW);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  float* Tp = reinterpret_cast<float*>(smem + Tile::BUF);  // KC x 32 NA plain t rows
  __shared__ __align__(8) uint64_t mma_done;
  __shared__ uint32_t tmem_slot;
  __shared__ int fptr[KC + 1], fmid[KC];
  __shared__ int sl[kNS];
  __shared__ float sv[kNS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  int i, f0, f1, slot = -1;
  if (p.unit) {
    const int4 u = reinterpret_cast<const int4*>(p.unit)[blockIdx.x];
    i = u.x;
    f0 = u.y;
    f1 = u.z;
    slot = u.w;
  } else {
    i = p.slice0 + blockIdx.x;
    f0 = p.slice_ptr[i];
    f1 = p.slice_ptr[i + 1];
  }
  if (f0 >= f1) return;  // empty slice: Y was zeroed before the launch

  // zero both buffers once: padding rows/columns (a >= J_mid, b >= J_leaf) are never written again
  for (int o = threadIdx.x * 16; o < Tile::BUF; o += 256 * 16)
    *reinterpret_cast<float4*>(smem + o) = make_float4(0.f, 0.f, 0.f, 0.f);
  if (threadIdx.x == 0) {
    tc::mbar_init(&mma_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(&tmem_slot)),
                 "r"(Tile::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  int nx_ptr = 0, nx_mid = 0;
  if (threadIdx.x <= min(KC, f1 - f0)) {
    nx_ptr = __ldg(p.fib_ptr + f0 + threadIdx.x);
    if (threadIdx.x < min(KC, f1 - f0)) nx_mid = __ldg(p.fib_mid + f0 + threadIdx.x);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t sbase = tc::smem_u32(smem);

  // register accumulators: warp w drains TMEM lanes 32 (w % 4).. (D rows = mid index), columns
  // [16 NA (w / 4), 16 NA (w / 4 + 1)) (the warp's lane quarter is fixed by its rank in the warpgroup)
  float racc[16 * NA];
#pragma unroll
  for (int j = 0; j < 16 * NA; ++j) racc[j] = 0.f;
  const uint32_t tq = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(16 * NA * (warp >> 2));
  auto drain = [&]() {
#pragma unroll
    for (int q = 0; q < NA; ++q) {
      float v[16];
      tc::tmem_ld16(tq + (uint32_t)(16 * q), v);
      tc::tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 16; ++j) racc[16 * q + j] += v[j];
    }
  };
  int c = 0;
  for (int fc = f0; fc < f1; fc += KC, ++c) {
    const int nf = min(KC, f1 - fc);
    uint8_t* buf = smem;
    uint8_t *Ahi = buf, *Alo = buf + TC_A_BYTES, *Bhi = buf + 2 * TC_A_BYTES,
            *Blo = buf + 2 * TC_A_BYTES + Tile::B_BYTES;
    if (threadIdx.x <= nf) fptr[threadIdx.x] = nx_ptr;
    if (threadIdx.x < nf) fmid[threadIdx.x] = nx_mid;
    __syncthreads();
    const int E0 = fptr[0], E1 = fptr[nf];
    const bool staged = E1 - E0 <= kNS;
    if (staged)
      for (int e = E0 + (int)threadIdx.x; e < E1; e += 256) {
        sl[e - E0] = __ldg(p.leaf_id + e);
        sv[e - E0] = __ldg(p.val + e);
      }
    const int fn = fc + KC;
    if (fn < f1) {
      const int nfn = min(KC, f1 - fn);
      if (threadIdx.x <= nfn) nx_ptr = __ldg(p.fib_ptr + fn + threadIdx.x);
      if (threadIdx.x < nfn) nx_mid = __ldg(p.fib_mid + fn + threadIdx.x);
    }
    __syncthreads();
    // leaf stage: warp per fiber -> row fl of the plain t buffer Tp (16-byte
    // chunks XOR-swizzled by fl & 7: conflict-free row stores and column reads)
    for (int fl = warp; fl < KC; fl += 8) {
      float t[QV][VW];
#pragma unroll
      for (int q = 0; q < QV; ++q)
#pragma unroll
        for (int k = 0; k < VW; ++k) t[q][k] = 0.f;
      if (fl < nf) {
        const int e0 = fptr[fl], e1 = fptr[fl + 1];
        int l[4];
        float x[4];
        if (staged) {
          for (int e = e0; e < e1; e += 4) {
            const int n = min(4, e1 - e);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              l[u] = u < n ? sl[e + u - E0] : 0;
              x[u] = u < n ? sv[e + u - E0] : 0.f;
            }
            gather_rows<VW, QV, 4>(l, x, n, p.Uleaf, p.ldl, p.Jl, lane, t);
          }
        } else {
          for (int e = e0; e < e1; e += 4) {
            const int n = min(4, e1 - e);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              l[u] = u < n ? __ldg(p.leaf_id + e + u) : 0;
              x[u] = u < n ? __ldg(p.val + e + u) : 0.f;
            }
            gather_rows<VW, QV, 4>(l, x, n, p.Uleaf, p.ldl, p.Jl, lane, t);
          }
        }
      }
      float* row = Tp + fl * (32 * NA);
#pragma unroll
      for (int q = 0; q < QV; ++q) {
        const int col = (lane + 32 * q) * VW;  // VW consecutive columns inside one 16-byte chunk
        if (col < 32 * NA) {
          const int pc = ((col >> 2) ^ (fl & 7)) * 4 + (col & 3);
          if constexpr (VW == 4) *reinterpret_cast<float4*>(row + pc) = make_float4(t[q][0], t[q][1], t[q][2], t[q][3]);
          else if constexpr (VW == 2) *reinterpret_cast<float2*>(row + pc) = make_float2(t[q][0], t[q][1]);
          else row[pc] = t[q][0];
        }
      }
    }
    // the operand buffer was last read by the MMAs of chunk c - 1; when c - 1 closed a TMEM
    // group, its sum moves into the registers before chunk c restarts the accumulator
    if (c >= 1) tc::mbar_wait(&mma_done, (uint32_t)((c - 1) & 1));
    if (c >= 1 && c % kTcGroup == 0) {
      tc::tc_fence_after();
      drain();
      tc::tc_fence_before();
    }
    __syncthreads();
    // transpose into the K-major operands: lanes run over the 32 fibers, so a
    // warp's store fills one 128-byte swizzle row (conflict-free)
    {
      const int k = lane;
      // B: rows n (leaf index), 4 per item, read as one 16-byte chunk of Tp row k
      for (int q = warp; q < 8 * NA; q += 8) {
        const float4 v = *reinterpret_cast<const float4*>(Tp + k * (32 * NA) + ((q ^ (k & 7)) << 2));
        st_split1(Bhi, Blo, k_sw128(4 * q, k), v.x);
        st_split1(Bhi, Blo, k_sw128(4 * q + 1, k), v.y);
        st_split1(Bhi, Blo, k_sw128(4 * q + 2, k), v.z);
        st_split1(Bhi, Blo, k_sw128(4 * q + 3, k), v.w);
      }
      // A: rows a (mid index) straight from the U_mid rows of the chunk's fibers
      if (k < nf) {
        const float* mr = p.Umid + (int64_t)fmid[k] * p.ldm;
        for (int a = warp; a < p.Jm; a += 8) st_split1(Ahi, Alo, k_sw128(a, k), __ldg(mr + a));
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      tc::tc_fence_after();
      const uint32_t ah = sbase, al = ah + TC_A_BYTES;
      const uint32_t bh = ah + 2 * TC_A_BYTES, bl = bh + Tile::B_BYTES;
#pragma unroll
      for (int g = 0; g < KC / 8; ++g) {
        const uint32_t o = (uint32_t)(g * 32);  // 8 tf32 = 32 bytes along K inside the swizzle row
        tc::umma_tf32(tmem, tc::sw128_desc(ah + o), tc::sw128_desc(bh + o), Tile::IDESC,
                      (c % kTcGroup > 0 || g > 0) ? 1u : 0u);
        tc::umma_tf32(tmem, tc::sw128_desc(ah + o), tc::sw128_desc(bl + o), Tile::IDESC, 1u);
        tc::umma_tf32(tmem, tc::sw128_desc(al + o), tc::sw128_desc(bh + o), Tile::IDESC, 1u);
      }
      tc::umma_commit(&mma_done);
    }
  }
  // all MMAs done once the last chunk's commit arrives; the last (partial) group joins the registers
  tc::mbar_wait(&mma_done, (uint32_t)((c - 1) & 1));
  tc::tc_fence_after();
  drain();
  {
    const int a = 32 * (warp & 3) + lane;  // D row = mid index
    if (a < p.Jm) {
#pragma unroll
      for (int j = 0; j < 16 * NA; ++j) {
        const int bcol = 16 * NA * (warp >> 2) + j;
        if (bcol < p.Jl) {
          if (slot >= 0) {
            p.part[(int64_t)slot * p.Jm * p.Jl + a * p.Jl + bcol] = racc[j];
          } else {
            const int64_t col = (p.a0 + a) * p.sa + (p.b0 + bcol) * p.sb;
            const int64_t off = p.transposed ? col * p.ldY + i : (int64_t)i * p.ldY + col;
            split_store(p.Yhi, p.Ylo, off, racc[j]);
          }
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Tile::TMEM_COLS));
}

// Y row of a split slice = sum of its units' partial tiles, in slot order
__global__ void __launch_bounds__(256) k_spttmc3_reduce(const int32_t* __restrict__ red,
                                                        const float* __restrict__ part, int Jm, int Jl,
                                                        int64_t sa, int64_t sb, float* Yhi, float* Ylo,
                                                        int64_t ldY, int transposed, int a0, int b0) {
  const int r = blockIdx.y;
  const int i = red[3 * r], s0 = red[3 * r + 1], ns = red[3 * r + 2];
  const int P = Jm * Jl;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= P) return;
  float y = 0.f;
  for (int s = 0; s < ns; ++s) y += __ldcs(part + (int64_t)(s0 + s) * P + c);
  const int a = c / Jl, b = c - a * Jl;
  const int64_t col = (a0 + a) * sa + (b0 + b) * sb;
  const int64_t off = transposed ? col * ldY + i : (int64_t)i * ldY + col;
  split_store(Yhi, Ylo, off, y);
}

struct Ttmc4Args {
  const int32_t *slice_ptr, *node_ptr, *node_mid0, *fib_ptr, *fib_mid1, *leaf_id;
  const float* val;
  const float *U0, *U1, *Uleaf;
  int J0, J1, Jl;
  float *Yhi, *Ylo;
  int64_t ldY;
  int transposed;
  int64_t s0, s1, sb;  // Kolda strides of (mid0, mid1, leaf) indices
  int slice0;          // first slice of this launch (rank shard) when unit == null
  const int32_t* unit; // work units (slice, node0, node1, slot) or null: one CTA per slice
  float* part;         // partial rows of split slices (J0 J1 Jl floats per slot)
  // k_spttmc4w: factor table sizes, padded strides and the cluster split of a slice
  int I_leaf, I_mid1;
  int J1P, J0P;        // J1, J0 rounded up to 4 (smem row strides)
  int csize;           // CTAs (cluster ranks) per slice
};

// ---------------------------------------------------------------------------
// Order-4 HOOI SpTTMc, node per warp (k_spttmc4w).  Per slice i (root) and
// node v = (i, mid0 index a):
//   leaf     t_f   = sum_{x in f} x U_leaf[leaf(x), :]          (Eq. 1; lanes = fibers)
//   level 2  Z_v   = sum_{f in v} U_mid1[mid1(f), :] (x) t_f     (J1 x Jl, lanes own 4x4 blocks)
//   level 3  Y_i  += U_mid0[a, :] (x) Z_v                        (all threads, per batch of 8 nodes)
// Each warp works on its own node (no block barrier inside a node); the CTA
// syncs twice per batch of 8 nodes for level 3.  U_leaf and U_mid1 are staged
// in shared memory when they fit (config 4: 16 KB each), zero padded to 4-float
// rows so every gather is a 128-bit load.  A slice is split over the `csize`
// CTAs of one thread-block cluster (contiguous node ranges); their partial Y
// rows are summed through distributed shared memory in fixed rank order
// (deterministic, no atomics, no partial rows in HBM) and written once.
// ---------------------------------------------------------------------------
constexpr int kW4 = 8;        // warps = nodes in flight per CTA
constexpr int kNPW = 1;       // nodes per warp between the CTA's level-3 barriers (2: one CTA per SM, slower)
constexpr int kB4 = kW4 * kNPW;  // nodes per batch
constexpr int kStage4 = 128;  // staged nonzeros per warp and fiber chunk (longer chunks read global memory)

// per-warp region (floats): T 32 x JLP | Z kNPW x (J1 x Jl <= J1P JLP) | bix 32 | staged leaf ids / values
__host__ __device__ inline int w4_floats(int JLP, int J1P) { return 32 * JLP + kNPW * J1P * JLP + 32 + 2 * kStage4; }

template <int JLP, int NBL, bool SM>
__global__ void __launch_bounds__(256, 2) k_spttmc4w(Ttmc4Args p) {
  extern __shared__ __align__(16) float sm4[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int J0 = p.J0, J1 = p.J1, Jl = p.Jl, J1P = p.J1P, J0P = p.J0P;
  const int P1 = J1 * Jl, P = J0 * P1;
  // layout: [U_leaf | U_mid1] (SM) | y (P, the slice's partial row) | u0t (J0P x kW4) | warp regions
  float* Uls = sm4;
  float* U1s = Uls + (SM ? p.I_leaf * JLP : 0);
  float* ys = U1s + (SM ? p.I_mid1 * J1P : 0);
  float* u0t = ys + ((P + 3) & ~3);
  float* wreg = u0t + J0P * kB4;
  const int WF = w4_floats(JLP, J1P);
  float* T = wreg + warp * WF;        // 32 x JLP fiber sums t_f
  float* Zr = T + 32 * JLP;           // kNPW node results, each J1 x Jl (compact, row j1)
  int* bix = reinterpret_cast<int*>(Zr + kNPW * J1P * JLP);
  int* stl = bix + 32;                // staged leaf ids
  float* stv = reinterpret_cast<float*>(stl + kStage4);
  const unsigned full = 0xffffffffu;

  const int csize = p.csize;
  const int slice = p.slice0 + (int)(blockIdx.x / csize);
  const int rank = (int)(blockIdx.x % csize);
  const int sn0 = p.slice_ptr[slice], sn1 = p.slice_ptr[slice + 1];
  const int n0 = sn0 + (int)((int64_t)(sn1 - sn0) * rank / csize);
  const int n1 = sn0 + (int)((int64_t)(sn1 - sn0) * (rank + 1) / csize);

  if (SM) {  // factor tables, rows zero padded to JLP / J1P floats
    for (int e = threadIdx.x; e < p.I_leaf * JLP; e += blockDim.x) {
      const int r = e / JLP, j = e - r * JLP;
      Uls[e] = j < Jl ? __ldg(p.Uleaf + (int64_t)r * Jl + j) : 0.f;
    }
    for (int e = threadIdx.x; e < p.I_mid1 * J1P; e += blockDim.x) {
      const int r = e / J1P, j = e - r * J1P;
      U1s[e] = j < J1 ? __ldg(p.U1 + (int64_t)r * J1 + j) : 0.f;
    }
  }
  for (int e = threadIdx.x; e < P; e += blockDim.x) ys[e] = 0.f;
  const int NB = (J1P / 4) * (JLP / 4);  // 4x4 blocks of Z
  // lane's Z blocks
  // (lanes past the last block compute on block 0 and never store: no branch in the fiber loop)
  int bro[NBL], bco[NBL];
  bool bon[NBL];
#pragma unroll
  for (int r = 0; r < NBL; ++r) {
    const int blk = lane + 32 * r;
    bon[r] = blk < NB;
    bro[r] = bon[r] ? 4 * (blk / (JLP / 4)) : 0;
    bco[r] = bon[r] ? 4 * (blk % (JLP / 4)) : 0;
  }
  __syncthreads();

  for (int base = n0; base < n1; base += kB4) {
   for (int h = 0; h < kNPW; ++h) {
    const int slot = h * kW4 + warp;  // the node's index in the batch
    const int nd = base + slot;
    float* Z = Zr + h * J1P * JLP;
    if (nd < n1) {
      float acc[NBL][4][4];
#pragma unroll
      for (int r = 0; r < NBL; ++r)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[r][i][j] = 0.f;
      const int f0 = __ldg(p.node_ptr + nd), f1 = __ldg(p.node_ptr + nd + 1);
      // chunk metadata one chunk ahead
      int eb = 0, ee = 0, b = 0;
      if (lane < min(32, f1 - f0)) {
        eb = __ldg(p.fib_ptr + f0 + lane);
        ee = __ldg(p.fib_ptr + f0 + lane + 1);
        b = __ldg(p.fib_mid1 + f0 + lane);
      }
      for (int fc = f0; fc < f1; fc += 32) {
        const int nf = min(32, f1 - fc);
        const int E0 = __shfl_sync(full, eb, 0), E1 = __shfl_sync(full, ee, nf - 1);
        const bool staged = E1 - E0 <= kStage4;
        if (staged) {
          for (int e = E0 + lane; e < E1; e += 32) {
            stl[e - E0] = __ldg(p.leaf_id + e);
            stv[e - E0] = __ldg(p.val + e);
          }
        }
        const int ceb = eb, cee = ee;
        bix[lane] = SM ? b * J1P : b;
        const int fn = fc + 32;
        eb = ee = b = 0;  // lanes past the next chunk's fibers: empty
        if (fn < f1 && lane < min(32, f1 - fn)) {
          eb = __ldg(p.fib_ptr + fn + lane);
          ee = __ldg(p.fib_ptr + fn + lane + 1);
          b = __ldg(p.fib_mid1 + fn + lane);
        }
        __syncwarp();
        float t[JLP];
#pragma unroll
        for (int j = 0; j < JLP; ++j) t[j] = 0.f;
        for (int e = ceb; e < cee; ++e) {  // lanes >= nf have ceb == cee
          int cl;
          float x;
          if (staged) {
            cl = stl[e - E0];
            x = stv[e - E0];
          } else {
            cl = __ldg(p.leaf_id + e);
            x = __ldg(p.val + e);
          }
          if (SM) {
            const float4* r4 = reinterpret_cast<const float4*>(Uls + cl * JLP);
#pragma unroll
            for (int q = 0; q < JLP / 4; ++q) {
              const float4 g = r4[q];
              t[4 * q] = fmaf(x, g.x, t[4 * q]);
              t[4 * q + 1] = fmaf(x, g.y, t[4 * q + 1]);
              t[4 * q + 2] = fmaf(x, g.z, t[4 * q + 2]);
              t[4 * q + 3] = fmaf(x, g.w, t[4 * q + 3]);
            }
          } else {
            const float* rg = p.Uleaf + (int64_t)cl * Jl;
#pragma unroll
            for (int j = 0; j < JLP; ++j)
              if (j < Jl) t[j] = fmaf(x, __ldg(rg + j), t[j]);
          }
        }
        float4* Tw = reinterpret_cast<float4*>(T + lane * JLP);
#pragma unroll
        for (int q = 0; q < JLP / 4; ++q) Tw[q] = make_float4(t[4 * q], t[4 * q + 1], t[4 * q + 2], t[4 * q + 3]);
        __syncwarp();
        // level 2: lane owns 4x4 blocks (rows j1 = bro.., cols jl = bco..) of Z; two fibers per step
        auto kron = [&](int k) {
          const int bk = bix[k];
#pragma unroll
          for (int r = 0; r < NBL; ++r) {
            {
              float4 u;
              if (SM) {
                u = *reinterpret_cast<const float4*>(U1s + bk + bro[r]);
              } else {
                const float* ug = p.U1 + (int64_t)bk * J1;
                const int j = bro[r];
                u.x = j < J1 ? __ldg(ug + j) : 0.f;
                u.y = j + 1 < J1 ? __ldg(ug + j + 1) : 0.f;
                u.z = j + 2 < J1 ? __ldg(ug + j + 2) : 0.f;
                u.w = j + 3 < J1 ? __ldg(ug + j + 3) : 0.f;
              }
              const float4 tt = *reinterpret_cast<const float4*>(T + k * JLP + bco[r]);
              const float ua[4] = {u.x, u.y, u.z, u.w}, ta[4] = {tt.x, tt.y, tt.z, tt.w};
#pragma unroll
              for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[r][i][j] = fmaf(ua[i], ta[j], acc[r][i][j]);
            }
          }
        };
        int k = 0;
        for (; k + 1 < nf; k += 2) {
          kron(k);
          kron(k + 1);
        }
        if (k < nf) kron(k);
        __syncwarp();  // T / bix / stage are rewritten by the next chunk
      }
      // node result Z (compact J1 x Jl) and its U_mid0 row (transposed: u0t[j0][warp])
#pragma unroll
      for (int r = 0; r < NBL; ++r) {
        if (bon[r]) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int j1 = bro[r] + i, jl = bco[r] + j;
              if (j1 < J1 && jl < Jl) Z[j1 * Jl + jl] = acc[r][i][j];
            }
        }
      }
      const float* ur = p.U0 + (int64_t)__ldg(p.node_mid0 + nd) * J0;
      for (int j = lane; j < J0P; j += 32) u0t[j * kB4 + slot] = j < J0 ? __ldg(ur + j) : 0.f;
    } else {
      for (int j = lane; j < J0P; j += 32) u0t[j * kB4 + slot] = 0.f;  // no node: zero weight
      for (int e = lane; e < J1 * Jl; e += 32) Z[e] = 0.f;
    }
   }
    __syncthreads();
    // level 3: y[j0, rem] += sum_w U_mid0[a_w, j0] Z_w[rem] over the batch's nodes; the thread's
    // positions rem keep the batch's Z values in registers, the weights come as broadcast loads
    for (int rem = threadIdx.x; rem < P1; rem += blockDim.x) {
      float z[kB4];
#pragma unroll
      for (int h = 0; h < kNPW; ++h)
#pragma unroll
        for (int w = 0; w < kW4; ++w) z[h * kW4 + w] = wreg[w * WF + 32 * JLP + h * J1P * JLP + rem];
      for (int j0 = 0; j0 < J0; ++j0) {
        const float4* a4 = reinterpret_cast<const float4*>(u0t + j0 * kB4);
        float sacc = ys[j0 * P1 + rem];
#pragma unroll
        for (int q = 0; q < kB4 / 4; ++q) {
          const float4 a = a4[q];
          sacc = fmaf(a.x, z[4 * q], sacc);
          sacc = fmaf(a.y, z[4 * q + 1], sacc);
          sacc = fmaf(a.z, z[4 * q + 2], sacc);
          sacc = fmaf(a.w, z[4 * q + 3], sacc);
        }
        ys[j0 * P1 + rem] = sacc;
      }
    }
    __syncthreads();
  }

  // cluster reduction of the slice's partial rows through distributed shared memory
  cg::cluster_group cl = cg::this_cluster();
  if (csize > 1) cl.sync();
  const int c0 = (int)((int64_t)P * rank / csize), c1 = (int)((int64_t)P * (rank + 1) / csize);
  for (int c = c0 + (int)threadIdx.x; c < c1; c += blockDim.x) {
    float v = 0.f;
    for (int r = 0; r < csize; ++r) {
      const float* peer = csize > 1 ? cl.map_shared_rank(ys, r) : ys;
      v += peer[c];
    }
    const int j0 = c / P1, rem = c - j0 * P1;
    const int j1 = rem / Jl, jl = rem - j1 * Jl;
    const int64_t col = j0 * p.s0 + j1 * p.s1 + jl * p.sb;
    const int64_t off = p.transposed ? col * p.ldY + slice : (int64_t)slice * p.ldY + col;
    split_store(p.Yhi, p.Ylo, off, v);
  }
  if (csize > 1) cl.sync();  // peers' shared memory stays alive until every rank has read it
}

struct SpmmArgs {
  const int32_t *fib_ptr, *fib_root, *fib_mid0, *fib_mid1, *leaf_id;
  const float* val;
  const float* U;
  int J;
  int64_t nfib, I_mid1;
  float *Whi, *Wlo;
  int64_t ldW, col_off;
  int64_t s_lo, s_hi, s_all;  // slices (mid index) of this rank of s_all; W columns start at col_off for s_lo
  int I_leaf;                  // rows of U (k_spmm_w's shared-memory table)
};

// One lane per fiber (MP's leaf SpMM, Fig. 7 X_s U_m): t_f = sum_{x in f} x U[leaf(x), :]
// in registers, 4*QV columns per pass (U rows read as 128-bit vectors when 4 | J),
// then written split (hi, lo) into W's K-tile-major layout at row root(f), columns
// col_off + (slice(f) - s_lo) J + j.  Fibers are consecutive per warp, so a warp's
// leaf ids / values come from one contiguous CSF range.
constexpr int kSpW = 4;  // warps per k_spmm_w block
// SM: the factor table U (I_leaf x J) is staged in shared memory (dynamic; when it
// fits) -- the per-nonzero row gathers then come from shared memory instead of L1
constexpr int kSpNz = 128;  // staged nonzeros per warp batch (longer batches read global memory)
template <int QV, bool SM>
__global__ void __launch_bounds__(32 * kSpW, 6) k_spmm_w(SpmmArgs p) {
  extern __shared__ __align__(16) float Us[];
  // per warp: 32 fibers x 4 QV split values of one column pass, then written out with
  // the warp's lanes over consecutive float4 slots: consecutive fibers of a CSF
  // ordering are consecutive slices of one row, i.e. consecutive W columns, so each
  // store instruction fills whole 128-byte K-tile row segments.  The batch's
  // nonzeros (leaf ids, values) are staged with coalesced loads, and the next
  // batch's fiber metadata is loaded while this batch computes.
  __shared__ __align__(16) float st4[kSpW][32 * 4 * QV];
  __shared__ int64_t srow[kSpW][32], scol[kSpW][32];
  __shared__ int snz_l[kSpW][kSpNz];
  __shared__ float snz_v[kSpW][kSpNz];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const bool sharded = p.s_lo > 0 || p.s_hi < p.s_all;
  const bool vec = (p.J & 3) == 0;                          // 128-bit U row loads
  const bool vst = vec && (p.col_off & 3) == 0;              // 128-bit W stores (4-aligned columns)
  const int64_t kt_stride = 32 * p.ldW;
  const int64_t nwarps = (int64_t)gridDim.x * kSpW;
  const float* Ub = p.U;
  if (SM) {
    const int n = p.I_leaf * p.J;
    for (int e = threadIdx.x; e < n; e += blockDim.x) Us[e] = __ldg(p.U + e);
    __syncthreads();
    Ub = Us;
  }
  struct Meta {
    int64_t mk, root;
    int e0, e1;
  };
  auto load_meta = [&](int64_t base) {
    Meta m{0, 0, 0, 0};
    const int64_t f = base + lane;
    if (f < p.nfib) {
      m.mk = __ldg(p.fib_mid0 + f);
      if (p.fib_mid1) m.mk = m.mk * p.I_mid1 + __ldg(p.fib_mid1 + f);
      m.root = __ldg(p.fib_root + f);
      m.e0 = __ldg(p.fib_ptr + f);
      m.e1 = __ldg(p.fib_ptr + f + 1);
    } else {
      m.e0 = m.e1 = -1;
    }
    return m;
  };
  int64_t base = (blockIdx.x * kSpW + warp) * 32LL;
  Meta nx = load_meta(base);
  for (; base < p.nfib; base += nwarps * 32) {
    const Meta cm = nx;
    nx = load_meta(base + nwarps * 32);  // in flight during this batch
    bool ok = cm.e0 >= 0 && !(sharded && (cm.mk < p.s_lo || cm.mk >= p.s_hi));
    // the batch's nonzeros [E0, E1) (contiguous in the CSF) staged with coalesced loads
    const int last = __popc(__ballot_sync(full, cm.e0 >= 0)) - 1;
    const int E0 = __shfl_sync(full, cm.e0, 0), E1 = __shfl_sync(full, cm.e1, last);
    const bool staged = E1 - E0 <= kSpNz;
    if (staged)
      for (int e = E0 + lane; e < E1; e += 32) {
        snz_l[warp][e - E0] = __ldg(p.leaf_id + e);
        snz_v[warp][e - E0] = __ldg(p.val + e);
      }
    const int e0 = ok ? cm.e0 : 0, e1 = ok ? cm.e1 : 0;
    const int64_t c0 = p.col_off + (cm.mk - p.s_lo) * p.J;
    srow[warp][lane] = ok ? cm.root : -1;
    scol[warp][lane] = c0;
    __syncwarp();
    for (int jb = 0; jb < p.J; jb += 4 * QV) {
      float t[4 * QV];
#pragma unroll
      for (int j = 0; j < 4 * QV; ++j) t[j] = 0.f;
      for (int e = e0; e < e1; e += 2) {
        const bool two = e + 1 < e1;
        float xa, xb;
        int la, lb;
        if (staged) {
          xa = snz_v[warp][e - E0];
          la = snz_l[warp][e - E0];
          xb = two ? snz_v[warp][e + 1 - E0] : 0.f;
          lb = two ? snz_l[warp][e + 1 - E0] : la;
        } else {
          xa = __ldg(p.val + e);
          la = __ldg(p.leaf_id + e);
          xb = two ? __ldg(p.val + e + 1) : 0.f;
          lb = two ? __ldg(p.leaf_id + e + 1) : la;
        }
        const float* ra = Ub + (int64_t)la * p.J + jb;
        const float* rb = Ub + (int64_t)lb * p.J + jb;
        if (vec) {
#pragma unroll
          for (int q = 0; q < QV; ++q) {
            if (jb + 4 * q < p.J) {
              const float4 g = SM ? reinterpret_cast<const float4*>(ra)[q] : __ldg(reinterpret_cast<const float4*>(ra) + q);
              const float4 k = SM ? reinterpret_cast<const float4*>(rb)[q] : __ldg(reinterpret_cast<const float4*>(rb) + q);
              t[4 * q] = fmaf(xb, k.x, fmaf(xa, g.x, t[4 * q]));
              t[4 * q + 1] = fmaf(xb, k.y, fmaf(xa, g.y, t[4 * q + 1]));
              t[4 * q + 2] = fmaf(xb, k.z, fmaf(xa, g.z, t[4 * q + 2]));
              t[4 * q + 3] = fmaf(xb, k.w, fmaf(xa, g.w, t[4 * q + 3]));
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < 4 * QV; ++j)
            if (jb + j < p.J) t[j] = fmaf(xb, rb[j], fmaf(xa, ra[j], t[j]));
        }
      }
      if (vst) {
        float4* t4 = reinterpret_cast<float4*>(st4[warp] + lane * 4 * QV);
#pragma unroll
        for (int q = 0; q < QV; ++q) t4[q] = make_float4(t[4 * q], t[4 * q + 1], t[4 * q + 2], t[4 * q + 3]);
        __syncwarp();
#pragma unroll
        for (int u = 0; u < QV; ++u) {
          const int slot = lane + 32 * u, k = slot / QV, q = slot - k * QV;
          const int64_t r = srow[warp][k];
          if (r >= 0 && jb + 4 * q < p.J) {
            const int64_t c = scol[warp][k] + jb + 4 * q;
            const int64_t off = (c >> 5) * kt_stride + r * 32 + (c & 31);
            const float4 v = reinterpret_cast<const float4*>(st4[warp])[slot];
            const float vv[4] = {v.x, v.y, v.z, v.w};
            float h[4], l[4];
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              h[w] = tf32_rna(vv[w]);
              l[w] = tf32_rna(vv[w] - h[w]);
            }
            *reinterpret_cast<float4*>(p.Whi + off) = make_float4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<float4*>(p.Wlo + off) = make_float4(l[0], l[1], l[2], l[3]);
          }
        }
        __syncwarp();
      } else if (ok) {
#pragma unroll
        for (int j = 0; j < 4 * QV; ++j) {
          if (jb + j < p.J) {
            const int64_t c = c0 + jb + j;
            split_store(p.Whi, p.Wlo, (c >> 5) * kt_stride + cm.root * 32 + (c & 31), t[j]);
          }
        }
      }
    }
    __syncwarp();
  }
}

inline int rtile(int J) { return (J + 15) / 16; }  // 1..8

// MP leaf SpMM for wide factor rows (J > 24) or factor tables too large for shared memory
// (config 2: U 1000 x 50 = 200 KB): lanes over the J columns instead of lane per fiber, so the
// U row gathers are coalesced (one 128-byte line per 32 columns of a row) and each store
// instruction writes 32 consecutive W columns of one row (one K-tile row segment).  A warp takes
// 32 consecutive fibers (metadata loaded coalesced, broadcast by shuffles) and walks them four
// at a time so four fibers' gathers are in flight together.
constexpr int kSpC = 8;  // warps per block
__global__ void __launch_bounds__(32 * kSpC) k_spmm_wc(SpmmArgs p) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const bool sharded = p.s_lo > 0 || p.s_hi < p.s_all;
  const int64_t kt_stride = 32 * p.ldW;
  const int64_t nwarps = (int64_t)gridDim.x * kSpC;
  for (int64_t base = (blockIdx.x * (int64_t)kSpC + warp) * 32; base < p.nfib; base += nwarps * 32) {
    const int64_t f = base + lane;
    int64_t mk = 0, root = -1;
    int e0 = 0, e1 = 0;
    if (f < p.nfib) {
      mk = __ldg(p.fib_mid0 + f);
      if (p.fib_mid1) mk = mk * p.I_mid1 + __ldg(p.fib_mid1 + f);
      root = __ldg(p.fib_root + f);
      e0 = __ldg(p.fib_ptr + f);
      e1 = __ldg(p.fib_ptr + f + 1);
      if (sharded && (mk < p.s_lo || mk >= p.s_hi)) e1 = e0 = 0, root = -1;
    }
    const int nf = (int)(p.nfib - base < 32 ? p.nfib - base : 32);
    for (int k0 = 0; k0 < nf; k0 += 4) {
      int ke0[4], ke1[4];
      int64_t kr[4], kc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kk = min(k0 + u, 31);
        ke0[u] = __shfl_sync(full, e0, kk);
        ke1[u] = k0 + u < nf ? __shfl_sync(full, e1, kk) : ke0[u];
        kr[u] = __shfl_sync(full, root, kk);
        kc[u] = p.col_off + (__shfl_sync(full, mk, kk) - p.s_lo) * p.J;
      }
      for (int jb = 0; jb < p.J; jb += 32) {
        const int j = jb + lane;
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        int lmax = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) lmax = max(lmax, ke1[u] - ke0[u]);
        for (int t = 0; t < lmax; ++t) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (t < ke1[u] - ke0[u]) {
              const int e = ke0[u] + t;
              const int l = __ldg(p.leaf_id + e);
              const float x = __ldg(p.val + e);
              if (j < p.J) acc[u] = fmaf(x, __ldg(p.U + (int64_t)l * p.J + j), acc[u]);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (k0 + u < nf && kr[u] >= 0 && j < p.J) {
            const int64_t c = kc[u] + j;
            split_store(p.Whi, p.Wlo, (c >> 5) * kt_stride + kr[u] * 32 + (c & 31), acc[u]);
          }
        }
      }
    }
  }
}

}  // namespace

// Kolda stride of mode `m` among the modes `others` (ascending lower-fastest).
static int64_t kolda_stride(int m, const int* others, int nothers, const int64_t* J) {
  int64_t s = 1;
  for (int k = 0; k < nothers; ++k)
    if (others[k] < m) s *= J[others[k]];
  return s;
}

// Mode c.mid0 from the Z kept by mode c.root's projection (spttmc4g.cu, k_spttmc4_sib)
void spttmc_hooi_sibling(const Csf& c, const float* Z, const float* const* U, const int64_t* J, Split out,
                         bool transposed, cudaStream_t st) {
  int others[3], no = 0;
  for (int m = 0; m < c.order; ++m)
    if (m != c.mid0) others[no++] = m;
  spttmc4_sibling(c, Z, U[c.root], J, out, transposed, kolda_stride(c.root, others, no, J),
                  kolda_stride(c.mid1, others, no, J), kolda_stride(c.leaf, others, no, J), st);
}

void spttmc_hooi(const Csf& c, const float* const* U, const int64_t* J, Split out, bool transposed,
                 cudaStream_t st, int64_t lo, int64_t hi, float* zout) {
  if (hi < 0) hi = c.I_root;
  if (hi <= lo) return;  // empty shard: Y stays zero
  int others[3], no = 0;
  for (int m = 0; m < c.order; ++m)
    if (m != c.root) others[no++] = m;
  const int64_t ldY = out.ld;
  if (c.order == 3) {
    Ttmc3Args a;
    a.slice_ptr = c.slice_ptr.p;
    a.fib_ptr = c.fib_ptr.p;
    a.fib_mid = c.fib_mid0.p;
    a.leaf_id = c.leaf_id.p;
    a.val = c.val.p;
    a.Umid = U[c.mid0];
    a.Uleaf = U[c.leaf];
    a.Jm = (int)J[c.mid0];
    a.Jl = (int)J[c.leaf];
    a.Yhi = out.hi;
    a.Ylo = out.lo;
    a.ldY = ldY;
    a.transposed = transposed;
    a.sa = kolda_stride(c.mid0, others, no, J);
    a.sb = kolda_stride(c.leaf, others, no, J);
    a.unit = c.nunits > 0 ? c.unit.p : nullptr;
    a.slice0 = (int)lo;  // the work plan (if any) was built for [lo, hi) already
    if (c.nunits > 0) {  // virtual fibers
      a.fib_ptr = c.vfib_ptr.p;
      a.fib_mid = c.vfib_mid.p;
    }
    a.part = c.part.p;
    const int RA = rtile(a.Jm), RB = rtile(a.Jl);
    const dim3 g((unsigned)(c.nunits > 0 ? c.nunits : hi - lo));
    bool launched = false;
    // U_leaf row vector width: rows of Jl floats are 16-byte aligned iff 4 | Jl
    const int VW = a.Jl % 4 == 0 ? 4 : (a.Jl % 2 == 0 ? 2 : 1);
    // tcgen05 Kronecker stage where the Kronecker work dominates (measured on
    // B200: J_mid J_leaf = 10^4 -> 35 vs 41 ms at config 5 mode 3; at 5000 and
    // 2500 the SIMT kernel's higher occupancy hides the gathers better: 35 vs
    // 42 ms, 0.28 vs 0.31 ms).  TUCKER_TTMC=tc|simt forces one (tests).
    const char* fe = std::getenv("TUCKER_TTMC");
    const int force = !fe ? 0 : (std::strcmp(fe, "tc") == 0 ? 1 : (std::strcmp(fe, "simt") == 0 ? -1 : 0));
    a.ldm = a.Jm;
    a.ldl = a.Jl;
    a.a0 = a.b0 = 0;
    const bool wide = a.Jm > 128 || a.Jl > 128;  // tcgen05 in 128 x 128 column windows
    const bool use_tc = wide || (force == 1 || (force == 0 && (int64_t)a.Jm * a.Jl >= 8192));
    const int Jm_full = a.Jm, Jl_full = a.Jl;
    const float* Umid_full = a.Umid;
    const float* Uleaf_full = a.Uleaf;
    for (int a0 = 0; use_tc && a0 < Jm_full; a0 += 128)
     for (int b0 = 0; b0 < Jl_full; b0 += 128) {
      a.a0 = a0;
      a.b0 = b0;
      a.Jm = std::min(128, Jm_full - a0);
      a.Jl = std::min(128, Jl_full - b0);
      a.Umid = Umid_full + a0;
      a.Uleaf = Uleaf_full + b0;
      launched = false;
      const int NA = (a.Jl + 31) / 32;
      const int VW = (Jl_full % 4 == 0 && b0 % 4 == 0) ? 4 : (Jl_full % 2 == 0 ? 2 : 1);
#define TK_TC(na, vw)                                                                          \
  if (!launched && NA == na && VW == vw) {                                                     \
    smem_optin((const void*)k_spttmc3_tc<na, vw>, TcTile<na>::SMEM);                          \
    TK_LAUNCH((k_spttmc3_tc<na, vw>), g, 256, TcTile<na>::SMEM, st, a);                        \
    launched = true;                                                                           \
  }
      TK_TC(1, 1) TK_TC(1, 2) TK_TC(1, 4) TK_TC(2, 1) TK_TC(2, 2) TK_TC(2, 4)
      TK_TC(3, 1) TK_TC(3, 2) TK_TC(3, 4) TK_TC(4, 1) TK_TC(4, 2) TK_TC(4, 4)
#undef TK_TC
      if (!launched) fail(TUCKER_E_ARG, "spttmc: no tcgen05 instance for this core size");
      if (c.nred > 0) {  // split slices: this window's partial tiles, summed in slot order
        const dim3 gr((unsigned)ceil_div((int64_t)a.Jm * a.Jl, 256), (unsigned)c.nred);
        TK_LAUNCH(k_spttmc3_reduce, gr, 256, 0, st, c.red.p, c.part.p, a.Jm, a.Jl, a.sa, a.sb, a.Yhi, a.Ylo, ldY,
                  (int)transposed, a0, b0);
      }
    }
    if (use_tc) {
      a.a0 = a.b0 = 0;
      a.Jm = Jm_full;
      a.Jl = Jl_full;
      a.Umid = Umid_full;
      a.Uleaf = Uleaf_full;
    }
#define TK_S3V(ra, rb, vw) \
  if (VW == vw) TK_LAUNCH((k_spttmc3<ra, rb, vw>), g, 256, 0, st, a);
#define TK_S3(ra, rb)                                                         \
  if (!launched && RA <= ra && RB <= rb) {                                     \
    TK_S3V(ra, rb, 1) TK_S3V(ra, rb, 2) TK_S3V(ra, rb, 4)                      \
    launched = true;                                                           \
  }
    // (8, 1): J_mid in (64, 128] with J_leaf <= 16 (config 3 mode 2: 100 x 10) -- without it the
    // dispatch fell through to (8, 2) and did twice the Kronecker FMAs on zero-padded columns
    TK_S3(1, 1) TK_S3(2, 1) TK_S3(1, 2) TK_S3(2, 2) TK_S3(4, 1) TK_S3(1, 4) TK_S3(4, 2)
    TK_S3(2, 4) TK_S3(4, 4) TK_S3(8, 1) TK_S3(8, 2) TK_S3(2, 8) TK_S3(8, 4) TK_S3(4, 8) TK_S3(8, 8)
#undef TK_S3
#undef TK_S3V
    if (!launched) fail(TUCKER_E_ARG, "spttmc: unsupported core size");
    if (c.nred > 0 && !use_tc) {
      const dim3 gr((unsigned)ceil_div((int64_t)a.Jm * a.Jl, 256), (unsigned)c.nred);
      TK_LAUNCH(k_spttmc3_reduce, gr, 256, 0, st, c.red.p, c.part.p, a.Jm, a.Jl, a.sa, a.sb, a.Yhi,
                a.Ylo, ldY, (int)transposed, 0, 0);
    }
    return;
  }
  Ttmc4Args a;
  a.slice_ptr = c.slice_ptr.p;
  a.node_ptr = c.node_ptr.p;
  a.node_mid0 = c.node_mid0.p;
  a.fib_ptr = c.fib_ptr.p;
  a.fib_mid1 = c.fib_mid1.p;
  a.leaf_id = c.leaf_id.p;
  a.val = c.val.p;
  a.U0 = U[c.mid0];
  a.U1 = U[c.mid1];
  a.Uleaf = U[c.leaf];
  a.J0 = (int)J[c.mid0];
  a.J1 = (int)J[c.mid1];
  a.Jl = (int)J[c.leaf];
  a.Yhi = out.hi;
  a.Ylo = out.lo;
  a.ldY = ldY;
  a.transposed = transposed;
  a.s0 = kolda_stride(c.mid0, others, no, J);
  a.s1 = kolda_stride(c.mid1, others, no, J);
  a.sb = kolda_stride(c.leaf, others, no, J);
  if (!std::getenv("TUCKER_TTMC4_CS") && !std::getenv("TUCKER_TTMC4_GMEM") &&
      spttmc4g(c, U, J, out, transposed, a.s0, a.s1, a.sb, st, lo, hi, zout))
    return;
  if (zout) fail(TUCKER_E_STATE, "spttmc_hooi: Z is kept by the GEMM-form kernel only");
  const int64_t P = (int64_t)a.J0 * a.J1 * a.Jl;
  a.slice0 = (int)lo;
  a.I_leaf = (int)c.I_leaf;
  a.I_mid1 = (int)c.I_mid1;
  a.J1P = (int)round_up(a.J1, 4);
  a.J0P = (int)round_up(a.J0, 4);
  const int JLP = (int)round_up(a.Jl, 4);
  const int NB = (a.J1P / 4) * (JLP / 4);
  const int64_t nsl = hi - lo;
  // cluster split: enough CTAs for ~4 per SM, at most 8 (portable cluster size)
  int num_sms = 0, dev = 0;
  TK_CUDA(cudaGetDevice(&dev));
  TK_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
  int cs = 1;
  while (cs < 8 && nsl * cs < 4 * num_sms) cs *= 2;
  if (const char* e = std::getenv("TUCKER_TTMC4_CS")) cs = std::max(1, std::min(8, std::atoi(e)));  // tests
  a.csize = cs;
  const size_t fac_bytes = ((size_t)a.I_leaf * JLP + (size_t)a.I_mid1 * a.J1P) * sizeof(float);
  const size_t rest_bytes = ((size_t)round_up(P, 4) + (size_t)a.J0P * kB4 + (size_t)kW4 * w4_floats(JLP, a.J1P)) *
                            sizeof(float);
  bool fac_smem = fac_bytes + rest_bytes <= 110 * 1024;
  if (std::getenv("TUCKER_TTMC4_GMEM")) fac_smem = false;  // tests: factors read from global memory
  const size_t smem = (fac_smem ? fac_bytes : 0) + rest_bytes;
  if (smem > 220 * 1024) fail(TUCKER_E_ARG, "spttmc: order-4 core too large for shared memory");
  bool launched = false;
  auto launch = [&](const void* fn) {
    smem_optin(fn, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(nsl * cs));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    void* args[] = {&a};
    TK_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
    if (g_launch_counter) ++(*g_launch_counter);
    if (sync_check_enabled()) TK_CUDA(cudaStreamSynchronize(st));
    launched = true;
  };
#define TK_S4W(jlp, nbl)                                                      \
  if (!launched && JLP == jlp && NB <= 32 * nbl) {                             \
    if (fac_smem) launch((const void*)k_spttmc4w<jlp, nbl, true>);             \
    else launch((const void*)k_spttmc4w<jlp, nbl, false>);                     \
  }
#define TK_S4WJ(jlp) TK_S4W(jlp, 1) TK_S4W(jlp, 2) TK_S4W(jlp, 4)
  TK_S4WJ(4) TK_S4WJ(8) TK_S4WJ(12) TK_S4WJ(16) TK_S4WJ(20) TK_S4WJ(24) TK_S4WJ(28) TK_S4WJ(32)
#undef TK_S4WJ
#undef TK_S4W
  if (!launched)
    fail(TUCKER_E_ARG, "spttmc: unsupported order-4 core size (leaf J <= 32, J_mid1 J_leaf <= 2048)");
}

// Work plan for the order-3 HOOI kernel (see Csf).  lmax = 1024 nonzeros
// per virtual fiber (the extra Kronecker updates cost <= J_m/1024 of the
// fiber stage); cmax = max(2^22, total work / (16 * #SMs)).  Uniform configs
// 1-4 have short fibers and light slices: no plan, one CTA per slice.
// Config 5's Zipf head (a slice with 7e6 nonzeros in <= 5000 fibers) is what
// this is for.
// Exact (int64) plan statistics on the device, so the common no-plan case costs
// three numbers of D2H instead of the fiber pointers: out[0] = longest fiber,
// out[1] = total work sum_f (wf ceil(L/lmax) + wn L), out[2] = heaviest slice
// wf F_i + wn nnz_i, over the slices [lo, hi).
__global__ void k_plan_stats(const int32_t* __restrict__ sp, const int32_t* __restrict__ fp, int64_t lo,
                             int64_t hi, int64_t lmax, int64_t wf, int64_t wn,
                             unsigned long long* __restrict__ out) {
  const int64_t f0 = sp[lo], f1 = sp[hi];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long lmx = 0, tot = 0, smx = 0;
  for (int64_t f = f0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < f1; f += stride) {
    const int64_t L = fp[f + 1] - fp[f];
    lmx = max(lmx, (unsigned long long)L);
    tot += (unsigned long long)(wf * ((L + lmax - 1) / lmax) + wn * L);
  }
  for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi; i += stride)
    smx = max(smx, (unsigned long long)(wf * (sp[i + 1] - sp[i]) + wn * (fp[sp[i + 1]] - fp[sp[i]])));
  atomicMax(out, lmx);
  atomicAdd(out + 1, tot);  // integer sum: order independent
  atomicMax(out + 2, smx);
}

void spttmc_plan(Csf& c, int64_t Jm, int64_t Jl, int num_sms, cudaStream_t st, int64_t lo, int64_t hi) {
  if (hi < 0) hi = c.I_root;
  if (c.order == 4) return;  // k_spttmc4w splits slices over thread-block clusters instead
  if (c.order != 3) return;
  const int64_t I = c.I_root, F = c.nfib;
  c.lmax = 1024;
  // test hooks: force the plan on small inputs (TUCKER_TTMC_LMAX / _CMAX)
  const char* el = std::getenv("TUCKER_TTMC_LMAX");
  const char* ec = std::getenv("TUCKER_TTMC_CMAX");
  if (el && std::atoll(el) > 0) c.lmax = std::atoll(el);
  const double wf = (double)Jm * Jl, wn = (double)Jl;  // work per fiber / per nonzero
  c.nunits = c.nred = c.nslots = c.nvfib = 0;
  if (hi <= lo) return;
  {
    DBuf<unsigned long long> stats(3);
    TK_CUDA(cudaMemsetAsync(stats.p, 0, 3 * sizeof(unsigned long long), st));
    TK_LAUNCH(k_plan_stats, 2 * num_sms, 256, 0, st, c.slice_ptr.p, c.fib_ptr.p, lo, hi, c.lmax, Jm * Jl, Jl,
              stats.p);
    unsigned long long h[3];
    TK_CUDA(cudaMemcpyAsync(h, stats.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaStreamSynchronize(st));
    c.cmax = std::max(4194304.0, (double)h[1] / (16.0 * num_sms));
    if (ec && std::atof(ec) > 0) c.cmax = std::atof(ec);
    if ((int64_t)h[0] <= c.lmax && (double)h[2] <= c.cmax) return;  // one CTA per slice
  }
  std::vector<int32_t> sp((size_t)I + 1), fp((size_t)F + 1);
  TK_CUDA(cudaMemcpyAsync(sp.data(), c.slice_ptr.p, sp.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaMemcpyAsync(fp.data(), c.fib_ptr.p, fp.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  std::vector<int32_t> fm((size_t)F);
  TK_CUDA(cudaMemcpyAsync(fm.data(), c.fib_mid0.p, fm.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  // virtual fibers, and per slice the virtual-fiber range
  std::vector<int32_t> vptr, vmid, vsp((size_t)I + 1);
  vptr.reserve((size_t)F + 1);
  vmid.reserve((size_t)F);
  for (int64_t i = lo; i < hi; ++i) {
    vsp[i] = (int32_t)vmid.size();
    for (int64_t f = sp[i]; f < sp[i + 1]; ++f) {
      const int64_t L = fp[f + 1] - fp[f], nv = std::max<int64_t>(1, ceil_div(L, c.lmax));
      for (int64_t v = 0; v < nv; ++v) {
        vptr.push_back((int32_t)(fp[f] + v * L / nv));
        vmid.push_back(fm[f]);
      }
    }
  }
  vsp[hi] = (int32_t)vmid.size();
  vptr.push_back(fp[sp[hi]]);
  c.nvfib = (int64_t)vmid.size();
  // units: greedy cut of each slice's virtual fibers at ~equal work
  std::vector<std::array<int32_t, 4>> units;
  std::vector<double> uw;
  std::vector<int32_t> red;
  int32_t slot = 0;
  for (int64_t i = lo; i < hi; ++i) {
    const int64_t v0 = vsp[i], v1 = vsp[i + 1];
    if (v1 == v0) continue;  // Y is zeroed before the launch
    const double w = wf * (double)(v1 - v0) + wn * (double)(vptr[v1] - vptr[v0]);
    if (w <= c.cmax) {
      units.push_back({(int32_t)i, (int32_t)v0, (int32_t)v1, -1});
      uw.push_back(w);
      continue;
    }
    const int64_t nu = (int64_t)std::ceil(w / c.cmax);
    const double target = w / (double)nu;
    const int32_t first = slot;
    int64_t a = v0;
    double acc = 0;
    for (int64_t v = v0; v < v1; ++v) {
      acc += wf + wn * (double)(vptr[v + 1] - vptr[v]);
      if (acc >= target || v + 1 == v1) {
        units.push_back({(int32_t)i, (int32_t)a, (int32_t)(v + 1), slot++});
        uw.push_back(acc);
        a = v + 1;
        acc = 0;
      }
    }
    red.insert(red.end(), {(int32_t)i, first, slot - first});
  }
  std::vector<int64_t> order(units.size());
  for (size_t u = 0; u < order.size(); ++u) order[u] = (int64_t)u;
  std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) { return uw[x] > uw[y]; });
  std::vector<int32_t> flat;
  flat.reserve(units.size() * 4);
  for (int64_t u : order) flat.insert(flat.end(), units[u].begin(), units[u].end());
  c.nunits = (int64_t)units.size();
  c.nred = (int64_t)red.size() / 3;
  c.nslots = slot;
  c.vfib_ptr.alloc(vptr.size());
  c.vfib_mid.alloc(vmid.size());
  c.unit.alloc(flat.size());
  TK_CUDA(cudaMemcpyAsync(c.vfib_ptr.p, vptr.data(), vptr.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  TK_CUDA(cudaMemcpyAsync(c.vfib_mid.p, vmid.data(), vmid.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  TK_CUDA(cudaMemcpyAsync(c.unit.p, flat.data(), flat.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  if (!red.empty()) {
    c.red.alloc(red.size());
    TK_CUDA(cudaMemcpyAsync(c.red.p, red.data(), red.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    c.part.alloc((size_t)(c.nslots * Jm * Jl));
  }
  TK_CUDA(cudaStreamSynchronize(st));  // the host vectors go out of scope
}

void spmm_mp(const Csf& c, const float* U_leaf, int64_t J_leaf, Split out, int64_t col_off,
             cudaStream_t st, int64_t s_lo, int64_t s_hi) {
  SpmmArgs a;
  a.s_all = c.I_mid0 * c.I_mid1;
  a.s_lo = s_lo;
  a.s_hi = s_hi < 0 ? a.s_all : s_hi;
  if (a.s_hi <= a.s_lo) return;
  a.fib_ptr = c.fib_ptr.p;
  a.fib_root = c.fib_root.p;
  a.fib_mid0 = c.fib_mid0.p;
  a.fib_mid1 = c.mid1 >= 0 ? c.fib_mid1.p : nullptr;
  a.leaf_id = c.leaf_id.p;
  a.val = c.val.p;
  a.U = U_leaf;
  a.J = (int)J_leaf;
  a.nfib = c.nfib;
  a.I_mid1 = c.I_mid1;
  a.Whi = out.hi;
  a.Wlo = out.lo;
  a.ldW = out.ld;
  a.col_off = col_off;
  if (!out.ktile) fail(TUCKER_E_ARG, "spmm_mp: W must be in the K-tile-major layout");
  a.I_leaf = (int)c.I_leaf;
  const size_t tab = (size_t)c.I_leaf * J_leaf * sizeof(float);
  const bool sm = tab <= 48 * 1024;
  int nsm = 148, dev = 0;
  TK_CUDA(cudaGetDevice(&dev));
  TK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  // persistent-ish grid (each block stages the table once), 6 blocks per SM
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(c.nfib, 32 * kSpW), 6 * std::max(1, nsm - g_sm_reserve)));
  const size_t smem = sm ? tab : 0;
  auto go = [&](const void* fn) {
    if (smem) smem_optin(fn, smem);
    void* args[] = {&a};
    TK_CUDA(cudaLaunchKernel(fn, dim3(blocks), dim3(32 * kSpW), args, smem, st));
    if (g_launch_counter) ++(*g_launch_counter);
    if (sync_check_enabled()) TK_CUDA(cudaStreamSynchronize(st));
  };
  if (J_leaf >= 32 && J_leaf <= 64 && !sm) {  // rows gathered from global memory: column lanes (k_spmm_wc;
    // measured: config 2 (J = 50) 0.85 -> ~0.2 ms per term; config 3 J = 100 keeps the lane-per-fiber kernel)
    const unsigned cblocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(c.nfib, 32 * kSpC),
                                                                            8 * std::max(1, nsm - g_sm_reserve)));
    TK_LAUNCH(k_spmm_wc, cblocks, 32 * kSpC, 0, st, a);
    return;
  }
#define TK_SPW(qv)                                         \
  if (sm) go((const void*)k_spmm_w<qv, true>);             \
  else go((const void*)k_spmm_w<qv, false>);
  if (J_leaf <= 8) { TK_SPW(2) }
  else if (J_leaf <= 16) { TK_SPW(4) }
  else if (J_leaf <= 24) { TK_SPW(6) }
  else { TK_SPW(8) }
#undef TK_SPW
}

}  // namespace tk
