// csf.cu -- COO validation and COO -> CSF (sorted slices/fibers) on the device.
//
// "To calculate the n-mode slices, we first sort the input
// tensor file by mode n ... After sorting on mode n, we can read the sorted file
// one slice at a time".  Here: one LSD radix sort of packed (root, mids, leaf)
// keys per ordering (CUB, one-time preprocessing inside tucker_init), then
// run-length boundaries give slice / node / fiber pointers.
#include <cub/cub.cuh>

#include <cstdlib>
#include <vector>
#include <algorithm>
#include <map>
#include <mutex>

#include "internal.cuh"

namespace tk {

thread_local int64_t* g_launch_counter = nullptr;
thread_local cudaStream_t g_alloc_stream = nullptr;
thread_local int g_sm_reserve = 0;
thread_local cudaEvent_t g_eig_kernel_event = nullptr;
void mempool_retain(int device) {
  static bool done[64] = {};
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  TK_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thr = ~0ull;
  TK_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  done[device] = true;
}

bool sync_check_enabled() {
  static const bool on = std::getenv("TUCKER_SYNC_CHECK") != nullptr;
  return on;
}

void smem_optin(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> set;
  int dev = 0;
  TK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = set[{fn, dev}];
  if (bytes <= cur) return;
  TK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  cur = bytes;
}

namespace {

__global__ void k_validate(int order, const int64_t* __restrict__ dims_unused, int64_t nnz,
                           const int32_t* __restrict__ i0, const int32_t* __restrict__ i1,
                           const int32_t* __restrict__ i2, const int32_t* __restrict__ i3,
                           int64_t d0, int64_t d1, int64_t d2, int64_t d3,
                           const float* __restrict__ v, int* flags, int32_t* keep) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    bool bad_idx = (i0[e] < 0 || i0[e] >= d0) || (i1[e] < 0 || i1[e] >= d1) ||
                   (order > 2 && (i2[e] < 0 || i2[e] >= d2)) ||
                   (order > 3 && (i3[e] < 0 || i3[e] >= d3));
    float x = v[e];
    bool bad_val = !isfinite(x);
    if (bad_idx) atomicOr(flags, 1);
    if (bad_val) atomicOr(flags, 2);
    keep[e] = (x != 0.0f) ? 1 : 0;  // explicit zeros are dropped
  }
}

__global__ void k_compact_i32(int64_t n, const int32_t* __restrict__ keep,
                              const int32_t* __restrict__ pos, const int32_t* __restrict__ in,
                              int32_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    if (keep[e]) out[pos[e]] = in[e];
}
__global__ void k_compact_f32(int64_t n, const int32_t* __restrict__ keep,
                              const int32_t* __restrict__ pos, const float* __restrict__ in,
                              float* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    if (keep[e]) out[pos[e]] = in[e];
}

// ||X||^2: per-block fp64 partials in a fixed grid, then one block sums them in order.
constexpr int kNormBlocks = 592;
__global__ void k_sumsq_partial(const float* __restrict__ v, int64_t n, double* part) {
  double s = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double x = v[e];
    s += x * x;
  }
  typedef cub::BlockReduce<double, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  double t = BR(tmp).Sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}
__global__ void k_sum_final(const double* part, int n, double* out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  typedef cub::BlockReduce<double, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  double t = BR(tmp).Sum(s);
  if (threadIdx.x == 0) *out = t;
}

__global__ void k_pack_keys(int64_t nnz, const int32_t* __restrict__ r, const int32_t* __restrict__ m0,
                            const int32_t* __restrict__ m1, const int32_t* __restrict__ lf,
                            int64_t I_m0, int64_t I_m1, int64_t I_leaf, uint64_t* __restrict__ key) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = (uint64_t)r[e];
    k = k * (uint64_t)I_m0 + (uint64_t)m0[e];
    if (m1) k = k * (uint64_t)I_m1 + (uint64_t)m1[e];
    k = k * (uint64_t)I_leaf + (uint64_t)lf[e];
    key[e] = k;
  }
}

// fiber flags: 1 where (root, mids) changes; duplicate detection on full keys.
__global__ void k_fiber_flags(int64_t nnz, const uint64_t* __restrict__ key, int64_t I_leaf,
                              int32_t* __restrict__ flag, int32_t* __restrict__ leaf_id, int* dup) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = key[e];
    leaf_id[e] = (int32_t)(k % (uint64_t)I_leaf);
    uint64_t fk = k / (uint64_t)I_leaf;
    int f = 1;
    if (e > 0) {
      uint64_t kp = key[e - 1];
      if (kp == k) atomicOr(dup, 1);
      f = (kp / (uint64_t)I_leaf) != fk;
    }
    flag[e] = f;
  }
}

__global__ void k_fiber_scatter(int64_t nnz, const uint64_t* __restrict__ key, int64_t I_leaf,
                                int64_t I_m0, int64_t I_m1, bool has_m1,
                                const int32_t* __restrict__ flag, const int32_t* __restrict__ pos,
                                int32_t* __restrict__ fib_ptr, int32_t* __restrict__ fib_root,
                                int32_t* __restrict__ fib_m0, int32_t* __restrict__ fib_m1) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[e]) continue;
    int32_t f = pos[e];
    uint64_t fk = key[e] / (uint64_t)I_leaf;
    fib_ptr[f] = (int32_t)e;
    if (has_m1) {
      fib_m1[f] = (int32_t)(fk % (uint64_t)I_m1);
      fk /= (uint64_t)I_m1;
    }
    fib_m0[f] = (int32_t)(fk % (uint64_t)I_m0);
    fib_root[f] = (int32_t)(fk / (uint64_t)I_m0);
  }
}

__global__ void k_node_flags(int64_t nfib, const int32_t* __restrict__ root,
                             const int32_t* __restrict__ m0, int32_t* __restrict__ flag) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nfib;
       f += (int64_t)gridDim.x * blockDim.x)
    flag[f] = (f == 0) || root[f] != root[f - 1] || m0[f] != m0[f - 1];
}
__global__ void k_node_scatter(int64_t nfib, const int32_t* __restrict__ flag,
                               const int32_t* __restrict__ pos, const int32_t* __restrict__ root,
                               const int32_t* __restrict__ m0, int32_t* __restrict__ node_ptr,
                               int32_t* __restrict__ node_root, int32_t* __restrict__ node_m0) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nfib;
       f += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[f]) continue;
    int32_t nd = pos[f];
    node_ptr[nd] = (int32_t)f;
    node_root[nd] = root[f];
    node_m0[nd] = m0[f];
  }
}

// slice_ptr[r] = first child whose root >= r (children sorted by root), r in [0, I_root]
__global__ void k_slice_ptr(int64_t I_root, const int32_t* __restrict__ child_root, int64_t nchild,
                            int32_t* __restrict__ slice_ptr) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= I_root;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nchild;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (child_root[mid] < r) lo = mid + 1; else hi = mid;
    }
    slice_ptr[r] = (int32_t)lo;
  }
}

__global__ void k_set_last(int32_t* p, int64_t i, int32_t v) { p[i] = v; }

inline int grid_for(int64_t n) {
  int64_t g = ceil_div(n, 256);
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

int bits_for(uint64_t total) {
  int b = 0;
  while (b < 64 && (total >> b) > 0) ++b;
  return b;
}

// exclusive scan of int32 flags into pos; returns total (sum of flags)
int64_t scan_flags(const int32_t* flag, int32_t* pos, int64_t n, DBuf<uint8_t>& tmp,
                   cudaStream_t st) {
  size_t bytes = 0;
  TK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, flag, pos, (int)n, st));
  tmp.ensure(bytes);
  TK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, flag, pos, (int)n, st));
  int32_t last_pos = 0, last_flag = 0;
  TK_CUDA(cudaMemcpyAsync(&last_pos, pos + n - 1, 4, cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaMemcpyAsync(&last_flag, flag + n - 1, 4, cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  return (int64_t)last_pos + last_flag;
}

}  // namespace

void coo_validate_compact(Coo& coo, cudaStream_t st) {
  const int64_t n = coo.nnz;
  DBuf<int> flags(1);
  DBuf<int32_t> keep(n), pos(n);
  TK_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int), st));
  const int32_t* ix[4] = {coo.idx[0].p, coo.idx[1].p, coo.order > 2 ? coo.idx[2].p : coo.idx[0].p,
                          coo.order > 3 ? coo.idx[3].p : coo.idx[0].p};
  TK_LAUNCH(k_validate, grid_for(n), 256, 0, st, coo.order, (const int64_t*)nullptr, n, ix[0], ix[1],
            ix[2], ix[3], coo.dims[0], coo.dims[1], coo.order > 2 ? coo.dims[2] : 1,
            coo.order > 3 ? coo.dims[3] : 1, coo.val.p, flags.p, keep.p);
  int h_flags = 0;
  TK_CUDA(cudaMemcpyAsync(&h_flags, flags.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  if (h_flags & 1) fail(TUCKER_E_INDEX, "tucker_init: an index is outside [0, I_n)");
  if (h_flags & 2) fail(TUCKER_E_VALUE, "tucker_init: non-finite value");
  DBuf<uint8_t> tmp;
  int64_t kept = scan_flags(keep.p, pos.p, n, tmp, st);
  if (kept == n) return;
  if (kept == 0) fail(TUCKER_E_VALUE, "tucker_init: all values are zero (||X|| = 0)");
  for (int m = 0; m < coo.order; ++m) {
    DBuf<int32_t> out(kept);
    TK_LAUNCH(k_compact_i32, grid_for(n), 256, 0, st, n, keep.p, pos.p, coo.idx[m].p, out.p);
    coo.idx[m] = std::move(out);
  }
  DBuf<float> vout(kept);
  TK_LAUNCH(k_compact_f32, grid_for(n), 256, 0, st, n, keep.p, pos.p, coo.val.p, vout.p);
  coo.val = std::move(vout);
  coo.nnz = kept;
  TK_CUDA(cudaStreamSynchronize(st));
}

double coo_norm2(const Coo& coo, cudaStream_t st) {
  DBuf<double> part(kNormBlocks), out(1);
  TK_LAUNCH(k_sumsq_partial, kNormBlocks, 256, 0, st, coo.val.p, coo.nnz, part.p);
  TK_LAUNCH(k_sum_final, 1, 256, 0, st, part.p, kNormBlocks, out.p);
  double h = 0;
  TK_CUDA(cudaMemcpyAsync(&h, out.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  return h;
}

void csf_build(const Coo& coo, Csf& c, int root, int mid0, int mid1, int leaf, cudaStream_t st) {
  const int64_t nnz = coo.nnz;
  c.order = coo.order;
  c.root = root;
  c.mid0 = mid0;
  c.mid1 = mid1;
  c.leaf = leaf;
  c.I_root = coo.dims[root];
  c.I_mid0 = coo.dims[mid0];
  c.I_mid1 = mid1 >= 0 ? coo.dims[mid1] : 1;
  c.I_leaf = coo.dims[leaf];
  c.nnz = nnz;
  const bool has_m1 = mid1 >= 0;

  DBuf<uint64_t> keys(nnz), keys_sorted(nnz);
  TK_LAUNCH(k_pack_keys, grid_for(nnz), 256, 0, st, nnz, coo.idx[root].p, coo.idx[mid0].p,
            has_m1 ? coo.idx[mid1].p : nullptr, coo.idx[leaf].p, c.I_mid0, c.I_mid1, c.I_leaf,
            keys.p);
  const uint64_t total = (uint64_t)c.I_root * (uint64_t)c.I_mid0 * (uint64_t)c.I_mid1 *
                         (uint64_t)c.I_leaf;
  const int end_bit = bits_for(total - 1 > 0 ? total - 1 : 1);
  c.val.alloc(nnz);
  DBuf<uint8_t> tmp;
  size_t bytes = 0;
  TK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, keys_sorted.p, coo.val.p, c.val.p,
                                          (int)nnz, 0, end_bit, st));
  tmp.ensure(bytes);
  TK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, keys.p, keys_sorted.p, coo.val.p, c.val.p,
                                          (int)nnz, 0, end_bit, st));
  if (g_launch_counter) ++(*g_launch_counter);
  keys.release();

  DBuf<int32_t> flag(nnz), pos(nnz);
  DBuf<int> dup(1);
  TK_CUDA(cudaMemsetAsync(dup.p, 0, sizeof(int), st));
  c.leaf_id.alloc(nnz);
  TK_LAUNCH(k_fiber_flags, grid_for(nnz), 256, 0, st, nnz, keys_sorted.p, c.I_leaf, flag.p,
            c.leaf_id.p, dup.p);
  int h_dup = 0;
  TK_CUDA(cudaMemcpyAsync(&h_dup, dup.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  const int64_t nfib = scan_flags(flag.p, pos.p, nnz, tmp, st);  // synchronises
  if (h_dup) fail(TUCKER_E_DUP, "tucker_init: duplicate coordinate");
  c.nfib = nfib;
  c.fib_ptr.alloc(nfib + 1);
  c.fib_root.alloc(nfib);
  c.fib_mid0.alloc(nfib);
  if (has_m1) c.fib_mid1.alloc(nfib);
  TK_LAUNCH(k_fiber_scatter, grid_for(nnz), 256, 0, st, nnz, keys_sorted.p, c.I_leaf, c.I_mid0,
            c.I_mid1, has_m1, flag.p, pos.p, c.fib_ptr.p, c.fib_root.p, c.fib_mid0.p,
            has_m1 ? c.fib_mid1.p : nullptr);
  TK_LAUNCH(k_set_last, 1, 1, 0, st, c.fib_ptr.p, nfib, (int32_t)nnz);
  keys_sorted.release();

  c.slice_ptr.alloc(c.I_root + 1);
  if (has_m1) {
    DBuf<int32_t> nflag(nfib), npos(nfib), node_root;
    TK_LAUNCH(k_node_flags, grid_for(nfib), 256, 0, st, nfib, c.fib_root.p, c.fib_mid0.p, nflag.p);
    const int64_t nnode = scan_flags(nflag.p, npos.p, nfib, tmp, st);
    c.nnode = nnode;
    c.node_ptr.alloc(nnode + 1);
    c.node_mid0.alloc(nnode);
    node_root.alloc(nnode);
    TK_LAUNCH(k_node_scatter, grid_for(nfib), 256, 0, st, nfib, nflag.p, npos.p, c.fib_root.p,
              c.fib_mid0.p, c.node_ptr.p, node_root.p, c.node_mid0.p);
    TK_LAUNCH(k_set_last, 1, 1, 0, st, c.node_ptr.p, nnode, (int32_t)nfib);
    TK_LAUNCH(k_slice_ptr, grid_for(c.I_root + 1), 256, 0, st, c.I_root, node_root.p, nnode,
              c.slice_ptr.p);
    TK_CUDA(cudaStreamSynchronize(st));
  } else {
    TK_LAUNCH(k_slice_ptr, grid_for(c.I_root + 1), 256, 0, st, c.I_root, c.fib_root.p, nfib,
              c.slice_ptr.p);
    TK_CUDA(cudaStreamSynchronize(st));
  }
}

}  // namespace tk

namespace tk {

// ---------------------------------------------------------------------------
// Sparse Gram S = X_(n) X_(n)^T for HO-SVD (Fig. 2, Fig. 4)
// and MP's pseudo HO-SVD (Fig. 7/8 P:921-937: (N-1) X_(n) X_(n)^T, the same
// eigenvectors).  c is an ordering whose LEAF is mode n, so one fiber = one
// column of X_(n) (all other indices fixed) with its leaf ids sorted.  Every
// fiber emits its pairs (i_a <= i_b, x_a x_b); a stable radix sort by the key
// i_a I + i_b and a reduce-by-key sum them in a fixed order (deterministic, no
// atomics); both triangles of S are then written.  Fibers [f0, f1) only (a
// rank's shard); S (fp64, row stride lds) must be zero beforehand.
// ---------------------------------------------------------------------------
namespace {

__global__ void k_pair_count(const int32_t* __restrict__ fib_ptr, int64_t f0, int64_t nf,
                             int64_t* __restrict__ cnt) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t L = fib_ptr[f0 + f + 1] - fib_ptr[f0 + f];
    cnt[f] = L * (L + 1) / 2;
  }
}

// warp per fiber: pairs (a, b >= a) in row-major triangle order
__global__ void k_pair_emit(const int32_t* __restrict__ fib_ptr, const int32_t* __restrict__ leaf,
                            const float* __restrict__ val, int64_t f0, int64_t nf,
                            const int64_t* __restrict__ off, int64_t base, int64_t I, int64_t* __restrict__ key,
                            double* __restrict__ pv) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t f = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; f < nf; f += nw) {
    const int64_t e0 = fib_ptr[f0 + f], L = fib_ptr[f0 + f + 1] - e0;
    int64_t o = off[f] - base;
    for (int64_t a = 0; a < L; ++a) {
      const int64_t ia = leaf[e0 + a];
      const double xa = (double)val[e0 + a];
      for (int64_t b = a + lane; b < L; b += 32) {
        key[o + (b - a)] = ia * I + leaf[e0 + b];
        pv[o + (b - a)] = xa * (double)val[e0 + b];
      }
      o += L - a;
    }
  }
}

__global__ void k_pair_scatter(const int64_t* __restrict__ ukey, const double* __restrict__ sum,
                               const int* __restrict__ nruns, int64_t I, double* __restrict__ S,
                               int64_t lds) {
  const int64_t n = *nruns;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = ukey[r] / I, j = ukey[r] - i * I;  // i <= j; keys unique within a chunk
    S[i * lds + j] += sum[r];
    if (i != j) S[j * lds + i] += sum[r];
  }
}

}  // namespace

void sparse_gram(const Csf& c, int64_t f0, int64_t f1, double* S, int64_t lds, cudaStream_t st) {
  const int64_t nf = f1 - f0, I = c.I_leaf;
  if (nf <= 0) return;
  DBuf<int64_t> cnt((size_t)nf + 1), off((size_t)nf + 1);
  TK_CUDA(cudaMemsetAsync(cnt.p + nf, 0, sizeof(int64_t), st));
  TK_LAUNCH(k_pair_count, grid_for(nf), 256, 0, st, c.fib_ptr.p, f0, nf, cnt.p);
  DBuf<uint8_t> tmp;
  size_t bytes = 0;
  TK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, off.p, nf + 1, st));
  tmp.ensure(bytes);
  TK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.p, off.p, nf + 1, st));
  // fibers in chunks of at most kPairChunk pairs (the sort's memory: 6 x 8 B per pair); each
  // chunk's pairs are sorted, reduced by key and added to S, chunks in fiber order
  // (deterministic).  A dense 10 % tensor (the paper's Table 2 at 1000^3) has 5e9 pairs per mode.
  constexpr int64_t kPairChunk = (int64_t)1 << 27;
  std::vector<int64_t> offh((size_t)nf + 1);
  TK_CUDA(cudaMemcpyAsync(offh.data(), off.p, offh.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  int64_t Pmax = 0;
  for (int64_t a = 0; a < nf;) {
    int64_t b = a + 1;
    while (b < nf && offh[b + 1] - offh[a] <= kPairChunk) ++b;
    Pmax = std::max(Pmax, offh[b] - offh[a]);
    a = b;
  }
  if (Pmax > ((int64_t)1 << 31) - 1)
    fail(TUCKER_E_OOM, "tucker_hosvd: one fiber of X_(n) has more than 2^31 pairs");
  DBuf<int64_t> key((size_t)Pmax), key2((size_t)Pmax), ukey((size_t)Pmax);
  DBuf<double> pv((size_t)Pmax), pv2((size_t)Pmax), sum((size_t)Pmax);
  DBuf<int> nruns(1);
  int bits = 1;
  while (((int64_t)1 << bits) < I * I) ++bits;
  for (int64_t a = 0; a < nf;) {
    int64_t b = a + 1;
    while (b < nf && offh[b + 1] - offh[a] <= kPairChunk) ++b;
    const int64_t P = offh[b] - offh[a];
    if (P > 0) {
      TK_LAUNCH(k_pair_emit, grid_for((b - a) * 32), 256, 0, st, c.fib_ptr.p, c.leaf_id.p, c.val.p, f0 + a, b - a,
                off.p + a, offh[a], I, key.p, pv.p);
      bytes = 0;
      TK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.p, key2.p, pv.p, pv2.p, (int)P, 0, bits, st));
      tmp.ensure(bytes);
      TK_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, key.p, key2.p, pv.p, pv2.p, (int)P, 0, bits, st));
      bytes = 0;
      TK_CUDA(cub::DeviceReduce::ReduceByKey(nullptr, bytes, key2.p, ukey.p, pv2.p, sum.p, nruns.p, cub::Sum(),
                                             (int)P, st));
      tmp.ensure(bytes);
      TK_CUDA(cub::DeviceReduce::ReduceByKey(tmp.p, bytes, key2.p, ukey.p, pv2.p, sum.p, nruns.p, cub::Sum(),
                                             (int)P, st));
      TK_LAUNCH(k_pair_scatter, grid_for(P), 256, 0, st, ukey.p, sum.p, nruns.p, I, S, lds);
    }
    a = b;
  }
  TK_CUDA(cudaStreamSynchronize(st));  // the scratch buffers go out of scope
}

}  // namespace tk
