// gen.cu -- HOOI's mode-n projection for tensor orders 2 and 5..8 (HOOI takes
// orders 2-8).  Fig. 4 is written for any N; order 2 is the matrix case of
// P:371-374 (Tucker = U S V^T).  Orders 3 and 4 -- every experiment of the paper, BASELINE's
// configs and MP's own scope -- keep the CSF kernels of spttmc*.cu; this path
// serves the remaining orders:
//   gen_build   per mode n, the nonzeros sorted by one 64-bit key (i_n most significant,
//               then the other modes with the lower mode fastest: prod_n I_n < 2^64 is checked
//               at init) with a device radix sort, and the slice pointers of mode n;
//               index / value validation, explicit zeros dropped, duplicates
//   spttmc_gen  Y_(n)[i_n, col] = sum_{x in slice i_n} x prod_{m != n} U_m[i_m, j_m(col)]
//               (Eq. 1 applied N - 1 times, Kolda column order, Eqs. 3-6): one CTA per slice,
//               threads over the columns, the slice's nonzeros staged in shared memory and
//               summed in their sorted order by every column (deterministic, no atomics).
// Correctness-first SIMT kernel (no fiber factoring): these orders are outside the paper's
// experiments and BASELINE's workloads.
#include <cub/cub.cuh>

#include <cstdint>

#include "internal.cuh"

namespace tk {
namespace {

__device__ __forceinline__ float tf32_rna_g(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

struct GenCooArgs {
  const int32_t* idx[kMaxOrder];
  int64_t dims[kMaxOrder];
  const float* val;
  int order;
  int64_t nnz;
};

// flags: 1 index out of range, 2 non-finite value; cnt: kept (nonzero) entries
__global__ void k_gen_validate(GenCooArgs a, int* flags, unsigned long long* cnt) {
  unsigned long long kept = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < a.nnz; e += (int64_t)gridDim.x * blockDim.x) {
    for (int m = 0; m < a.order; ++m) {
      const int32_t i = a.idx[m][e];
      if (i < 0 || i >= a.dims[m]) atomicOr(flags, 1);
    }
    const float v = a.val[e];
    if (!isfinite(v)) atomicOr(flags, 2);
    kept += v != 0.0f;
  }
  if (kept) atomicAdd(cnt, kept);
}

// key of mode n: i_n * S_n + sum_{m != n} i_m stride_m (lower modes fastest); zeros -> UINT64_MAX
__global__ void k_gen_key(GenCooArgs a, int n, uint64_t* key) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < a.nnz; e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t lin = 0, stride = 1;
    for (int m = 0; m < a.order; ++m) {
      if (m == n) continue;
      lin += (uint64_t)a.idx[m][e] * stride;
      stride *= (uint64_t)a.dims[m];
    }
    key[e] = a.val[e] != 0.0f ? (uint64_t)a.idx[n][e] * stride + lin : ~0ull;
  }
}

__global__ void k_gen_dup(const uint64_t* key, int64_t kept, int* flags) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; e < kept; e += (int64_t)gridDim.x * blockDim.x)
    if (key[e] == key[e - 1]) atomicOr(flags, 4);
}

// sptr[i] = first sorted entry with key >= i * Sn, i in [0, I_n]
__global__ void k_gen_sptr(const uint64_t* key, int64_t kept, uint64_t Sn, int64_t In, int32_t* sptr) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= In; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t t = (uint64_t)i * Sn;
    int64_t lo = 0, hi = kept;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (key[mid] < t) lo = mid + 1;
      else hi = mid;
    }
    sptr[i] = (int32_t)lo;
  }
}

constexpr int kGenT = 256;   // threads (columns in flight) per CTA
constexpr int kGenCh = 128;  // nonzeros staged per chunk

struct GenTtmcArgs {
  const uint64_t* key;
  const float* val;
  const int32_t* sptr;
  const float* U[kMaxOrder - 1];  // the other modes, ascending
  int J[kMaxOrder - 1];
  int64_t I[kMaxOrder - 1];
  uint64_t Sn;                    // prod_{m != n} I_m
  int64_t P;                      // prod_{m != n} J_m
  float *Yhi, *Ylo;
  int64_t ld;
  int transposed;
};

template <int NO>  // number of other modes (order - 1)
__global__ void __launch_bounds__(kGenT) k_spttmc_gen(GenTtmcArgs a) {
  __shared__ int32_t sidx[NO][kGenCh];
  __shared__ float sval[kGenCh];
  const int64_t i = blockIdx.x;
  const int e0 = a.sptr[i], e1 = a.sptr[i + 1];
  if (e0 == e1) return;  // empty slice: the row stays zero
  for (int64_t cb = 0; cb < a.P; cb += kGenT) {
    const int64_t col = cb + threadIdx.x;
    int jd[NO];
    {
      int64_t r = col;
#pragma unroll
      for (int q = 0; q < NO; ++q) {
        jd[q] = (int)(r % a.J[q]);
        r /= a.J[q];
      }
    }
    float acc = 0.0f;
    for (int c0 = e0; c0 < e1; c0 += kGenCh) {
      const int nch = min(kGenCh, e1 - c0);
      __syncthreads();
      for (int t = threadIdx.x; t < nch; t += kGenT) {
        uint64_t r = a.key[c0 + t] % a.Sn;
#pragma unroll
        for (int q = 0; q < NO; ++q) {
          sidx[q][t] = (int32_t)(r % (uint64_t)a.I[q]);
          r /= (uint64_t)a.I[q];
        }
        sval[t] = a.val[c0 + t];
      }
      __syncthreads();
      if (col < a.P)
        for (int t = 0; t < nch; ++t) {
          float p = sval[t];
#pragma unroll
          for (int q = 0; q < NO; ++q) p *= __ldg(a.U[q] + (int64_t)sidx[q][t] * a.J[q] + jd[q]);
          acc += p;
        }
    }
    if (col < a.P) {
      const int64_t off = a.transposed ? col * a.ld + i : i * a.ld + col;
      const float h = tf32_rna_g(acc);
      a.Yhi[off] = h;
      a.Ylo[off] = tf32_rna_g(acc - h);
    }
  }
}

inline unsigned gblocks(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 4096)); }

}  // namespace

void gen_build(Coo& coo, GenMode* modes, cudaStream_t st) {
  GenCooArgs a;
  for (int m = 0; m < kMaxOrder; ++m) {
    a.idx[m] = m < coo.order ? coo.idx[m].p : nullptr;
    a.dims[m] = m < coo.order ? coo.dims[m] : 1;
  }
  a.val = coo.val.p;
  a.order = coo.order;
  a.nnz = coo.nnz;
  DBuf<int> flags(1);
  DBuf<unsigned long long> cnt(1);
  TK_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int), st));
  TK_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
  TK_LAUNCH(k_gen_validate, gblocks(coo.nnz), 256, 0, st, a, flags.p, cnt.p);
  int hf = 0;
  unsigned long long kept = 0;
  TK_CUDA(cudaMemcpyAsync(&hf, flags.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaMemcpyAsync(&kept, cnt.p, sizeof(kept), cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  if (hf & 1) fail(TUCKER_E_INDEX, "tucker_init: an index is outside [0, I_n)");
  if (hf & 2) fail(TUCKER_E_VALUE, "tucker_init: non-finite value");
  if (kept == 0) fail(TUCKER_E_VALUE, "tucker_init: all values are zero (||X|| = 0)");
  DBuf<uint64_t> keys(coo.nnz);
  DBuf<uint8_t> tmp;
  for (int n = 0; n < coo.order; ++n) {
    GenMode& g = modes[n];
    TK_LAUNCH(k_gen_key, gblocks(coo.nnz), 256, 0, st, a, n, keys.p);
    g.key.alloc(coo.nnz);
    g.val.alloc(coo.nnz);
    size_t bytes = 0;
    TK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, g.key.p, coo.val.p, g.val.p, (int)coo.nnz, 0, 64, st));
    tmp.ensure(bytes);
    TK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, keys.p, g.key.p, coo.val.p, g.val.p, (int)coo.nnz, 0, 64, st));
    g.nnz = (int64_t)kept;
    uint64_t Sn = 1;
    for (int m = 0; m < coo.order; ++m)
      if (m != n) Sn *= (uint64_t)coo.dims[m];
    g.Sn = Sn;
    if (n == 0) {
      TK_LAUNCH(k_gen_dup, gblocks(g.nnz), 256, 0, st, g.key.p, g.nnz, flags.p);
      TK_CUDA(cudaMemcpyAsync(&hf, flags.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      TK_CUDA(cudaStreamSynchronize(st));
      if (hf & 4) fail(TUCKER_E_DUP, "tucker_init: duplicate coordinate");
    }
    g.sptr.alloc(coo.dims[n] + 1);
    TK_LAUNCH(k_gen_sptr, gblocks(coo.dims[n] + 1), 256, 0, st, g.key.p, g.nnz, Sn, coo.dims[n], g.sptr.p);
  }
  TK_CUDA(cudaStreamSynchronize(st));
}

void spttmc_gen(const GenMode& g, int order, int n, const int64_t* dims, const int64_t* J, const float* const* U,
                Split Y, bool transposed, cudaStream_t st) {
  GenTtmcArgs a;
  int q = 0;
  int64_t P = 1;
  for (int m = 0; m < order; ++m) {
    if (m == n) continue;
    a.U[q] = U[m];
    a.J[q] = (int)J[m];
    a.I[q] = dims[m];
    P *= J[m];
    ++q;
  }
  a.key = g.key.p;
  a.val = g.val.p;
  a.sptr = g.sptr.p;
  a.Sn = g.Sn;
  a.P = P;
  a.Yhi = Y.hi;
  a.Ylo = Y.lo;
  a.ld = Y.ld;
  a.transposed = transposed ? 1 : 0;
  const unsigned grid = (unsigned)dims[n];
  switch (order - 1) {
    case 1: TK_LAUNCH(k_spttmc_gen<1>, grid, kGenT, 0, st, a); break;
    case 2: TK_LAUNCH(k_spttmc_gen<2>, grid, kGenT, 0, st, a); break;
    case 3: TK_LAUNCH(k_spttmc_gen<3>, grid, kGenT, 0, st, a); break;
    case 4: TK_LAUNCH(k_spttmc_gen<4>, grid, kGenT, 0, st, a); break;
    case 5: TK_LAUNCH(k_spttmc_gen<5>, grid, kGenT, 0, st, a); break;
    case 6: TK_LAUNCH(k_spttmc_gen<6>, grid, kGenT, 0, st, a); break;
    case 7: TK_LAUNCH(k_spttmc_gen<7>, grid, kGenT, 0, st, a); break;
    default: fail(TUCKER_E_ARG, "spttmc_gen: order 2..8");
  }
}

}  // namespace tk
