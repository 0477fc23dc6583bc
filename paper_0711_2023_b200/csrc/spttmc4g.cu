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
  const int32_t* sp;        // slot nonzero offsets, SPC per (batch, chunk)
  const int32_t* leaf;      // nonzeros in slot order
  const float* val;
  const float *U0, *U1, *Ul;
  int J0, J1, Jl, JLP, J0P, CL, NB, NCH, SPC;
  int I_leaf, I_mid1;
  int b_lo, nb;             // batches [b_lo, b_lo + nb) of this launch
  float* part;              // [nb][J0 * J1 * JLP] partial rows of runs (index: run's first batch - b_lo)
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          tc::smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
      : "memory");
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
  const int SB = p.SPC + 2 * kCap;  // ints per stage buffer

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
    tc::mbar_expect_tx(&full[buf], (uint32_t)(p.SPC * 4 + (ok ? 8 * n : 0)));
    bulk_g2s(sb, p.sp + (ck0 + q) * p.SPC, (uint32_t)(p.SPC * 4), &full[buf]);
    if (ok && n > 0) {
      bulk_g2s(sb + p.SPC, p.leaf + E0r, (uint32_t)(4 * n), &full[buf]);
      bulk_g2s(sb + p.SPC + kCap, p.val + E0r, (uint32_t)(4 * n), &full[buf]);
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
        const int v = s % NB, bl = s / NB;
        float4 t[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) t[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int e = e0; e < e1; ++e) {
          int l;
          float x;
          if (ok) {
            l = sb[p.SPC + e - E0r];
            x = __int_as_float(sb[p.SPC + kCap + e - E0r]);
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
                           int NB, int SPC, int32_t* __restrict__ cnt, int32_t* __restrict__ fslot) {
  const int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f >= nfib) return;
  int64_t lo = 0, hi = nnode;
  while (hi - lo > 1) {
    const int64_t m = (lo + hi) / 2;
    if (node_ptr[m] <= f) lo = m;
    else hi = m;
  }
  const int b = fib_mid1[f];
  const int s = node_base[lo] + (b / kKCH) * SPC + (b % kKCH) * NB;
  cnt[s] = fib_ptr[f + 1] - fib_ptr[f];
  fslot[f] = s;
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
  return (size_t)(fl + 2 * (SPC + 2 * kCap)) * 4;
}

// Build (once per ordering) and run the GEMM-form SpTTMc; false = not applicable
// (caller falls back to k_spttmc4w).  TUCKER_TTMC4=w disables it, =g forces it
// (tests) where it fits at all.
bool spttmc4g(const Csf& c, const float* const* U, const int64_t* J, Split out, bool transposed, int64_t s0,
              int64_t s1, int64_t sb, cudaStream_t st, int64_t lo, int64_t hi) {
  const char* fe = std::getenv("TUCKER_TTMC4");
  const int force = !fe ? 0 : (fe[0] == 'g' ? 1 : (fe[0] == 'w' ? -1 : 0));
  if (force < 0 || c.order != 4) return false;
  const int J0 = (int)J[c.mid0], J1 = (int)J[c.mid1], Jl = (int)J[c.leaf];
  const int JLP = (int)round_up(Jl, 4), J1P = (int)round_up(J1, 4), CL = JLP / 4;
  if (J1P > 24 || CL > 8 || J0 > 256) return false;
  const int NB = kNT / CL;
  const int NCH = (int)ceil_div(c.I_mid1, kKCH);
  const int SPC = (int)round_up((int64_t)NB * kKCH + 1, 4);
  // density: slots (nodes x I_mid1, rounded to batches) against fibers
  const double slots_est = (double)c.nnode * (double)NCH * kKCH;
  if (force == 0 && slots_est > 2.5 * (double)c.nfib) return false;
  if (g4_smem(c, J0, J1, Jl, NB, SPC) > 220 * 1024) return false;

  Csf::G4& g = *c.g4;
  if (g.jlp != JLP) {  // build the dense batch layout
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
                c.fib_mid1.p, c.nfib, node_base.p, NB, SPC, cnt.p, fslot.p);
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
    g.jlp = JLP;
  }
  const int blo = g.bfirst_h[lo], bhi = g.bfirst_h[hi];
  const int nb = bhi - blo;
  if (nb <= 0) return true;  // empty shard: Y stays zero
  const int64_t P = (int64_t)J0 * J1 * JLP;
  g.part.ensure((size_t)nb * P);
  int nsm = 148, dev = 0;
  TK_CUDA(cudaGetDevice(&dev));
  TK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const int G = std::min(nb, nsm);
  G4Args a;
  a.batch = g.batch.p;
  a.node_mid0 = c.node_mid0.p;
  a.sp = g.sp.p;
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
  const dim3 gr((unsigned)ceil_div(P, 256), (unsigned)(hi - lo));
  TK_LAUNCH(k_spttmc4g_reduce, gr, 256, 0, st, (const float*)g.part.p, (const int32_t*)g.bfirst.p, (int)lo, blo, nb, G,
            J1, Jl, JLP, (int)P, s0, s1, sb, out.hi, out.lo, out.ld, (int)transposed);
  return true;
}

}  // namespace tk
