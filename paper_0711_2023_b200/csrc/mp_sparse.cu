// mp_sparse.cu -- MP's multislice Gram without the dense W (order 3, tensors whose
// W_n would not fit in HBM: BASELINE config 5, W_1 ~ 0.6 TB).
//
// Fig. 7 / Appendix: M_n = sum_{m != n} sum_s P_s P_s^T,
// P_s = X_s U_m, the slice s fixing the third mode o.  With the CSF ordering
// (root o, mid n, leaf m) the fibers of slice s are contiguous and sorted by their
// mode-n index i_n, and fiber f is one row of P_s:
//   P[f, :] = t_f = sum_{x in f} x U_m[leaf(x), :]                          (Eq. 1)
//   M_n[i(f), i(g)] += <P[f, :], P[g, :]>   for every pair of fibers f, g of one slice.
//
// k_mp_prows writes P (fp32, one row per fiber).  k_mp_slice_gram is a persistent
// cooperative kernel that walks the slices in order: the upper-triangle 128 x 128
// tiles of the slice's compact P_s P_s^T are spread over the CTAs, each a 3xTF32
// tcgen05 product (hi.hi + hi.lo + lo.hi, K = J_m <= 128, fp32 in TMEM) whose
// entries are added in fp64 to M_n at (i(f), i(g)) -- the upper triangle only,
// i(f) <= i(g) since a slice's fibers are sorted by i.  One grid barrier per slice
// orders the additions of different slices into the same entry: every entry
// receives its contributions in slice order (deterministic, no atomics).  The
// dense W path costs 2 d^2 sum_s J_m flops; this one 2 J_m sum_s r_s^2 (r_s =
// fibers of slice s) and r_s^2 / 2 fp64 read-modify-writes per slice.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "internal.cuh"
#include "tc_ptx.cuh"

namespace cg = cooperative_groups;

namespace tk {
namespace {

__device__ __forceinline__ float tf32r(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// one lane per fiber: P[f, 0..JP) = t_f (zero padded past J)
template <int QV>
__global__ void __launch_bounds__(256) k_mp_prows(const int32_t* __restrict__ fib_ptr,
                                                  const int32_t* __restrict__ leaf_id,
                                                  const float* __restrict__ val, const float* __restrict__ U,
                                                  int J, int JP, int64_t f0, int64_t f1, float* __restrict__ P) {
  const bool vec = (J & 3) == 0;
  for (int64_t f = f0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < f1;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int e0 = __ldg(fib_ptr + f), e1 = __ldg(fib_ptr + f + 1);
    float* out = P + (f - f0) * JP;
    for (int jb = 0; jb < JP; jb += 4 * QV) {
      float t[4 * QV];
#pragma unroll
      for (int j = 0; j < 4 * QV; ++j) t[j] = 0.f;
      for (int e = e0; e < e1; e += 2) {
        const bool two = e + 1 < e1;
        const float xa = __ldg(val + e), xb = two ? __ldg(val + e + 1) : 0.f;
        const int la = __ldg(leaf_id + e), lb = two ? __ldg(leaf_id + e + 1) : la;
        const float* ra = U + (int64_t)la * J + jb;
        const float* rb = U + (int64_t)lb * J + jb;
        if (vec) {
#pragma unroll
          for (int q = 0; q < QV; ++q)
            if (jb + 4 * q < J) {
              const float4 g = __ldg(reinterpret_cast<const float4*>(ra) + q);
              const float4 k = __ldg(reinterpret_cast<const float4*>(rb) + q);
              t[4 * q] = fmaf(xb, k.x, fmaf(xa, g.x, t[4 * q]));
              t[4 * q + 1] = fmaf(xb, k.y, fmaf(xa, g.y, t[4 * q + 1]));
              t[4 * q + 2] = fmaf(xb, k.z, fmaf(xa, g.z, t[4 * q + 2]));
              t[4 * q + 3] = fmaf(xb, k.w, fmaf(xa, g.w, t[4 * q + 3]));
            }
        } else {
#pragma unroll
          for (int j = 0; j < 4 * QV; ++j)
            if (jb + j < J) t[j] = fmaf(xb, __ldg(rb + j), fmaf(xa, __ldg(ra + j), t[j]));
        }
      }
#pragma unroll
      for (int q = 0; q < QV; ++q)
        if (jb + 4 * q < JP)
          *reinterpret_cast<float4*>(out + jb + 4 * q) =
              make_float4(t[4 * q], t[4 * q + 1], t[4 * q + 2], t[4 * q + 3]);
    }
  }
}

constexpr int NTH = 256;
constexpr int TT = 128;           // tile rows / cols
constexpr int KCH = 32;           // K per chunk (one 128-byte swizzle row)
constexpr int OPB = TT * KCH * 4; // one operand chunk (16 KB)
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TT >> 3) << 17) |
                           ((uint32_t)(TT >> 4) << 24);

struct SliceGramArgs {
  const float* P;              // fibers [fbase, ...) x JP, fp32
  const int32_t* rowid;        // mode-n index of each fiber (fib_mid0 of the (o, n, m) ordering)
  const int32_t* slice_ptr;    // fibers of slice s: [slice_ptr[s], slice_ptr[s + 1])
  int64_t fbase;               // first fiber held in P
  int s0, s1;                  // slices of this launch
  int J, JP, nkc;              // J_m, P's row stride, K chunks (JP rounded up to 32, / 32)
  double* M;                   // fp64 upper triangle, row stride ls
  int64_t ls;
};

// byte offset of element (row, k) in a K-major SW128 tile (32 K per row)
__device__ __forceinline__ uint32_t sw(int row, int k) {
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((((k >> 2) ^ (row & 7)) << 4) | ((k & 3) << 2)));
}

__global__ void __launch_bounds__(NTH, 1) k_mp_slice_gram(SliceGramArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* Ahi = sm;
  uint8_t* Alo = sm + OPB;
  uint8_t* Bhi = sm + 2 * OPB;
  uint8_t* Blo = sm + 3 * OPB;
  float* Ds = reinterpret_cast<float*>(sm + 4 * OPB);  // TT x (TT + 1) staged result
  __shared__ int Ra[TT], Rb[TT];
  __shared__ __align__(8) uint64_t mma_bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, cta = blockIdx.x;
  cg::grid_group grid = cg::this_grid();
  if (threadIdx.x == 0) {
    tc::mbar_init(&mma_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tslot)),
                 "r"(TT));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t sbase = tc::smem_u32(sm);
  uint32_t phase = 0;

  for (int s = p.s0; s < p.s1; ++s) {
    const int64_t fs = p.slice_ptr[s], fe = p.slice_ptr[s + 1];
    const int r = (int)(fe - fs);
    const int T = (r + TT - 1) / TT;
    const int ntile = T * (T + 1) / 2;
    // the slice's tiles over the CTAs, starting at a slice-dependent CTA so light slices spread out
    const int start = (int)(((int64_t)s * 37) % G);
    for (int t = (cta - start + G) % G; t < ntile; t += G) {
      // upper-triangle tile index -> (a, b), a <= b
      int a = 0, rem = t;
      while (rem >= T - a) {
        rem -= T - a;
        ++a;
      }
      const int b = a + rem;
      const bool diag = a == b;
      const int ra = min(TT, r - TT * a), rb = min(TT, r - TT * b);
      const int64_t ga = fs + (int64_t)TT * a - p.fbase, gb = fs + (int64_t)TT * b - p.fbase;
      if (threadIdx.x < TT) {
        Ra[threadIdx.x] = threadIdx.x < ra ? __ldg(p.rowid + fs + TT * a + threadIdx.x) : 0;
        Rb[threadIdx.x] = threadIdx.x < rb ? __ldg(p.rowid + fs + TT * b + threadIdx.x) : 0;
      }
      for (int kc = 0; kc < p.nkc; ++kc) {
        // stage the K chunk: row i of A (B) = P[ga (gb) + i, 32 kc ..], split into tf32 hi / lo
        for (int u = threadIdx.x; u < TT * (KCH / 4); u += NTH) {
          const int i = u >> 3, k4 = (u & 7) << 2, col = KCH * kc + k4;
          float4 va = make_float4(0.f, 0.f, 0.f, 0.f), vb = va;
          if (i < ra && col < p.JP) va = *reinterpret_cast<const float4*>(p.P + (ga + i) * p.JP + col);
          if (!diag && i < rb && col < p.JP) vb = *reinterpret_cast<const float4*>(p.P + (gb + i) * p.JP + col);
          const float xa[4] = {va.x, va.y, va.z, va.w}, xb[4] = {vb.x, vb.y, vb.z, vb.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t o = sw(i, k4 + q);
            const float h = tf32r(xa[q]);
            *reinterpret_cast<float*>(Ahi + o) = h;
            *reinterpret_cast<float*>(Alo + o) = tf32r(xa[q] - h);
            if (!diag) {
              const float hb = tf32r(xb[q]);
              *reinterpret_cast<float*>(Bhi + o) = hb;
              *reinterpret_cast<float*>(Blo + o) = tf32r(xb[q] - hb);
            }
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
          tc::tc_fence_after();
          const uint32_t ah = sbase, al = sbase + OPB;
          const uint32_t bh = diag ? ah : sbase + 2 * OPB, bl = diag ? al : sbase + 3 * OPB;
#pragma unroll
          for (int g = 0; g < KCH / 8; ++g) {
            const uint32_t o = (uint32_t)(g * 32);
            tc::umma_tf32(tmem, tc::sw128_desc(ah + o), tc::sw128_desc(bh + o), IDESC, (kc > 0 || g > 0) ? 1u : 0u);
            tc::umma_tf32(tmem, tc::sw128_desc(ah + o), tc::sw128_desc(bl + o), IDESC, 1u);
            tc::umma_tf32(tmem, tc::sw128_desc(al + o), tc::sw128_desc(bh + o), IDESC, 1u);
          }
          tc::umma_commit(&mma_bar);
        }
        tc::mbar_wait(&mma_bar, phase);  // the operands are rewritten by the next chunk
        phase ^= 1u;
        tc::tc_fence_after();
      }
      // D (row = A row, col = B row) -> shared memory, then fp64 adds with lanes over columns
      if (warp < 4) {
#pragma unroll
        for (int q = 0; q < TT / 32; ++q) {
          float v[32];
          tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(32 * q), v);
          tc::tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) Ds[(32 * warp + lane) * (TT + 1) + 32 * q + j] = v[j];
        }
      }
      tc::tc_fence_before();
      __syncthreads();
      for (int i = warp; i < ra; i += NTH / 32) {
        double* mrow = p.M + (int64_t)Ra[i] * p.ls;
        for (int c = lane; c < rb; c += 32)
          if (!diag || c >= i) mrow[Rb[c]] += (double)Ds[i * (TT + 1) + c];
      }
      __syncthreads();  // Ds / Ra / Rb are reused by the next tile
    }
    grid.sync();  // the next slice may add into the same entries
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TT));
}

// lower triangle = upper triangle (row-major, stride ls)
__global__ void k_mirror_upper(double* M, int64_t d, int64_t ls) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < d * d; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / d, j = e - i * d;
    if (i > j) M[i * ls + j] = M[j * ls + i];
  }
}

}  // namespace

size_t mp_sparse_smem() { return 4 * OPB + (size_t)TT * (TT + 1) * sizeof(float) + 1024; }

void mp_sparse_term(const Csf& c, const float* U_leaf, int64_t J, int64_t s_lo, int64_t s_hi, double* M, int64_t ls,
                    DBuf<float>& Pbuf, size_t max_p_floats, cudaStream_t st) {
  if (c.order != 3) fail(TUCKER_E_ARG, "mp_sparse_term: order 3 only");
  if (J > 128) fail(TUCKER_E_ARG, "mp_sparse_term: J_m <= 128");
  const int JP = (int)round_up(J, 4);
  const int nkc = (int)ceil_div(JP, KCH);
  std::vector<int32_t> sp((size_t)c.I_root + 1);
  TK_CUDA(cudaMemcpyAsync(sp.data(), c.slice_ptr.p, sp.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  if (s_hi < 0) s_hi = c.I_root;
  const size_t smem = mp_sparse_smem();
  smem_optin((const void*)k_mp_slice_gram, smem);
  int dev = 0, nsm = 148;
  TK_CUDA(cudaGetDevice(&dev));
  TK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  {
    int per = 0;
    TK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_mp_slice_gram, NTH, smem));
    if (per < 1) fail(TUCKER_E_CUDA, "k_mp_slice_gram cannot be resident");
  }
  // slices in batches whose P rows fit the buffer (one P pass + one Gram launch per batch)
  int64_t s = s_lo;
  while (s < s_hi) {
    int64_t e = s;
    while (e < s_hi && (size_t)(sp[e + 1] - sp[s]) * JP <= max_p_floats) ++e;
    if (e == s) fail(TUCKER_E_OOM, "mp_sparse_term: one slice's P rows exceed the buffer");
    const int64_t f0 = sp[s], f1 = sp[e];
    Pbuf.ensure((size_t)std::max<int64_t>(1, (f1 - f0) * JP));
    if (f1 > f0) {
      const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(f1 - f0, 256), 148 * 16);
      if (JP <= 32) TK_LAUNCH((k_mp_prows<8>), blocks, 256, 0, st, c.fib_ptr.p, c.leaf_id.p, c.val.p, U_leaf,
                              (int)J, JP, f0, f1, Pbuf.p);
      else TK_LAUNCH((k_mp_prows<8>), blocks, 256, 0, st, c.fib_ptr.p, c.leaf_id.p, c.val.p, U_leaf, (int)J, JP,
                     f0, f1, Pbuf.p);
      SliceGramArgs a;
      a.P = Pbuf.p;
      a.rowid = c.fib_mid0.p;
      a.slice_ptr = c.slice_ptr.p;
      a.fbase = f0;
      a.s0 = (int)s;
      a.s1 = (int)e;
      a.J = (int)J;
      a.JP = JP;
      a.nkc = nkc;
      a.M = M;
      a.ls = ls;
      void* args[] = {&a};
      TK_CUDA(cudaLaunchCooperativeKernel((const void*)k_mp_slice_gram, dim3(nsm), dim3(NTH), args, smem, st));
      if (g_launch_counter) ++(*g_launch_counter);
      if (sync_check_enabled()) TK_CUDA(cudaStreamSynchronize(st));
    }
    s = e;
  }
}

void mp_sparse_mirror(double* M, int64_t d, int64_t ls, cudaStream_t st) {
  const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(d * d, 256), 148 * 32);
  TK_LAUNCH(k_mirror_upper, blocks, 256, 0, st, M, d, ls);
}

}  // namespace tk
