// tucker.cu -- the C-ABI (include/tucker.h): handle, validation, and the
// per-sweep orchestration of the kernels in csf.cu / spttmc.cu / gram*.cu /
// eig.cu / dense.cu.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "internal.cuh"

using namespace tk;

struct tucker_handle {
  int order = 0;
  int64_t dims[kMaxOrder] = {1, 1, 1, 1, 1, 1, 1, 1};
  int64_t J[kMaxOrder] = {1, 1, 1, 1, 1, 1, 1, 1};
  tucker_opts opts{};
  cudaStream_t st = nullptr;
  bool own_stream = false;
  Coo coo;
  std::vector<std::unique_ptr<Csf>> csfs;
  int hooi_csf[kMaxOrder] = {-1, -1, -1, -1, -1, -1, -1, -1};
  bool generic = false;      // order 2 or 5..8: HOOI through gen.cu (no CSF, no MP / SP)
  GenMode gen[kMaxOrder];
  int mp_csf[kMaxOrder][kMaxOrder];
  DBuf<float> U[kMaxOrder];
  double normX2 = 0;
  // workspaces
  DBuf<float> Yhi, Ylo, Whi, Wlo;
  // W_n per (mode, term set): W's zero blocks depend only on the tensor, and the
  // SpMM rewrites every present block in full, so a kept buffer needs no memset
  // on later builds (kept while all handles' kept buffers fit a quarter of the
  // device memory)
  struct WKeep {
    DBuf<float> hi, lo;
    size_t need = 0;
  };
  WKeep wkeep[kMaxOrder][kMaxOrder + 1];
  size_t wkeep_bytes = 0;  // this handle's share of g_wkeep_bytes (returned when it is freed)
  ~tucker_handle();
  Split Y;  // last HOOI projection (mode Y_mode)
  int Y_mode = -1;
  bool Y_transposed = false;
  DBuf<double> S, V, Ufull, G64, scal;
  DBuf<float> Pmp;  // MP sparse multislice Gram: P rows of a batch of slices
  DBuf<float> G32, Ytmp;
  bool G_valid = false;
  EigSlot slots[3][kMaxOrder];  // warm starts: [0] HOOI, [1] MP, [2] SP
  double last_g2 = 0;           // ||G||_F^2 of the last core (SP's Delta_G rule)
  DBuf<double> theta_d;
  DBuf<int> info_d;                        // eigensolver info records (16 ints each)
  EigSlot* rec_slot[kMaxOrder + 1] = {};   // slot of each record: [n] sweep mode n, [kMaxOrder] one-off
  EigSlot scratch_slot;
  EigWs eig;
  GramWs gram;
  // MP overlap (mp_sweep): while mode n's eigensolve runs, a second stream builds the next
  // mode's W columns that do not involve U_n and their partial Gram into S2
  cudaStream_t st2 = nullptr, st_hi = nullptr;  // side work (least priority), eigensolve (greatest)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_eig = nullptr;
  DBuf<double> S2;
  GramWs gram2;
  bool side_ready[kMaxOrder] = {};
  cudaEvent_t tl[kMaxOrder][8] = {};  // TUCKER_MP_TIMELINE=1: fork, eig end, side SpMM end, side Gram end,
                                      // late start, late SpMM end, late Gram end
  int64_t launches = 0;
  int64_t stat_outer0 = 0, stat_matvec0 = 0, stat_sweeps0 = 0;
  long long prof0[13] = {0};
  std::string last_error;
  bool eig_unconverged = false;
  // multi-GPU: a sharded sweep when opts.nccl_unique_id is set
  void* comm = nullptr;
  bool sharded = false;
  int64_t hooi_lo[kMaxOrder] = {}, hooi_hi[kMaxOrder] = {-1, -1, -1, -1, -1, -1, -1, -1};  // root slices of mode n
  std::vector<int64_t> hooi_bounds[kMaxOrder];  // every rank's root-slice bounds of mode n (world + 1)
  int64_t mp_lo[kMaxOrder][kMaxOrder] = {}, mp_hi[kMaxOrder][kMaxOrder] = {};       // slices of MP term (n, m)
  bool Y_partial = false;  // h->Y holds only this rank's rows (Y^T Y route, not gathered)
  // HOOI partial-contraction reuse (order 4, one rank, GEMM-form SpTTMc): mode p's projection on the
  // ordering (p; p + 1; x; y) keeps Z = X x_x U_x^T x_y U_y^T per node (i_p, i_{p+1}); mode p + 1 is
  // then one small kernel over Z.  valid: Z was built with the current U_x and U_y.
  struct Memo {
    int csf = -1, root = -1, sib = -1;
    DBuf<float> Z;
    bool valid = false;
  };
  Memo memo[2];
  int64_t memo_hits = 0;
  // MP overlap accounting (tucker_mp_overlap_times): kernel time by stream, summed at each sweep's
  // end from the tl events.  [0] side SpMM, [1] side Gram, [2] late / whole SpMM (main stream),
  // [3] late / whole Gram, [4] eigensolve + factor (its own stream).  cnt: SpMM in terms (= launches),
  // the others in calls.
  double ov_ms[5] = {};
  int64_t ov_cnt[5] = {};
  unsigned tl_rec[kMaxOrder] = {};  // this sweep's recorded groups: 1 fork/eig, 2 side, 4 late
};
// kept W buffers of all live handles in this process (budget: a quarter of the device)
static std::atomic<size_t> g_wkeep_bytes{0};
tucker_handle::~tucker_handle() {
  g_wkeep_bytes -= wkeep_bytes;
  for (auto& row : tl)
    for (auto& e : row)
      if (e) cudaEventDestroy(e);
}


namespace {

struct SmReserveScope {  // SMs held by a concurrent kernel (MP overlap): grid sizing leaves them out
  int prev;
  explicit SmReserveScope(int n) : prev(g_sm_reserve) { g_sm_reserve = n; }
  ~SmReserveScope() { g_sm_reserve = prev; }
};

struct AllocScope {  // stream-ordered allocations on another stream of the handle (MP overlap)
  cudaStream_t prev;
  explicit AllocScope(cudaStream_t s) : prev(g_alloc_stream) { g_alloc_stream = s; }
  ~AllocScope() { g_alloc_stream = prev; }
};

struct LaunchScope {  // route TK_LAUNCH counting and stream-ordered allocations to this handle
  int64_t* prev;
  cudaStream_t prev_st;
  explicit LaunchScope(tucker_handle* h) : prev(g_launch_counter), prev_st(g_alloc_stream) {
    g_launch_counter = &h->launches;
    g_alloc_stream = h->st;
  }
  ~LaunchScope() {
    g_launch_counter = prev;
    g_alloc_stream = prev_st;
  }
};

template <typename F>
int guarded(tucker_handle* h, F&& f) {
  try {
    if (h) {
      LaunchScope ls(h);
      TK_CUDA(cudaSetDevice(h->opts.device));
      return f();
    }
    return f();
  } catch (const Error& e) {
    if (h) h->last_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    if (h) h->last_error = "host allocation failed";
    return TUCKER_E_OOM;
  } catch (const std::exception& e) {
    if (h) h->last_error = e.what();
    return TUCKER_E_CUDA;
  }
}

__global__ void k_combine(const float* __restrict__ hi, const float* __restrict__ lo, int64_t rows,
                          int64_t cols, int64_t ld, float* __restrict__ out) {
  const int64_t n = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols, c = e % cols;
    out[e] = hi[r * ld + c] + lo[r * ld + c];
  }
}
__global__ void k_scale_cols(double* V, int64_t d, int J, const double* __restrict__ s) {
  const int64_t n = d * J;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    V[e] *= s[e % J];
}
// V[:, j] *= theta_j^{-1/2} (0 if theta_j <= 0), theta on the device
__global__ void k_scale_cols_rsqrt(double* V, int64_t d, int J, const double* __restrict__ theta) {
  const int64_t n = d * J;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double t = theta[e % J];
    V[e] *= t > 0 ? 1.0 / sqrt(t) : 0.0;
  }
}
__global__ void k_d2f(const double* __restrict__ x, int64_t n, float* __restrict__ y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    y[e] = (float)x[e];
}
// ||G||^2 in fp64 (single CTA, fixed order) and Eq. 9 fit via the norm identity
__global__ void k_core_fit(const double* __restrict__ G, int64_t n, double normX2, double* out) {
  __shared__ double red[512];
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) s += G[e] * G[e];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 256; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double g2 = red[0];
    out[0] = g2;
    out[1] = 1.0 - sqrt(fmax(0.0, normX2 - g2)) / sqrt(normX2);
  }
}

inline int gridn(int64_t n) {
  int64_t g = ceil_div(n, 256);
  if (g > 148 * 8) g = 148 * 8;
  return (int)(g < 1 ? 1 : g);
}

int64_t prod_J_except(const tucker_handle* h, int n) {
  int64_t P = 1;
  for (int m = 0; m < h->order; ++m)
    if (m != n) P *= h->J[m];
  return P;
}

const float* const* uptrs(tucker_handle* h) {
  static thread_local const float* p[kMaxOrder];
  for (int m = 0; m < h->order; ++m) p[m] = h->U[m].p;
  return p;
}

// factor n was rewritten (n < 0: all): the kept Z products that used it are stale
void memo_invalidate(tucker_handle* h, int n) {
  for (auto& m : h->memo) {
    if (m.csf < 0) continue;
    const Csf& c = *h->csfs[m.csf];
    if (n < 0 || n == c.mid1 || n == c.leaf) m.valid = false;
  }
}

EigOpts eig_opts(const tucker_handle* h) {
  EigOpts o;
  o.oversample = h->opts.eig_oversample;
  if (h->opts.eig_max_iter > 0) o.max_outer = h->opts.eig_max_iter;
  else o.max_outer = 60;
  if (h->opts.eig_tol > 0) o.tol = h->opts.eig_tol;
  return o;
}

// Y_(n) (or its transpose) with the current factors into h->Y (split, zero padded)
void project_hooi(tucker_handle* h, int n, bool transposed) {
  const int64_t P = prod_J_except(h, n);
  const int64_t rows = transposed ? P : h->dims[n];
  const int64_t cols = transposed ? h->dims[n] : P;
  const int64_t rows_pad = round_up(rows, 128), ld = round_up(cols, 32);
  const size_t need = (size_t)(rows_pad * ld);
  h->Yhi.ensure(need);
  h->Ylo.ensure(need);
  TK_CUDA(cudaMemsetAsync(h->Yhi.p, 0, need * sizeof(float), h->st));
  TK_CUDA(cudaMemsetAsync(h->Ylo.p, 0, need * sizeof(float), h->st));
  h->Y.hi = h->Yhi.p;
  h->Y.lo = h->Ylo.p;
  h->Y.rows = rows;
  h->Y.cols = cols;
  h->Y.ld = ld;
  tucker_handle::Memo* mroot = nullptr;
  tucker_handle::Memo* msib = nullptr;
  for (auto& m : h->memo) {
    if (m.csf >= 0 && m.root == n) mroot = &m;
    if (m.csf >= 0 && m.sib == n && m.valid) msib = &m;
  }
  if (h->generic) {
    spttmc_gen(h->gen[n], h->order, n, h->dims, h->J, uptrs(h), h->Y, transposed, h->st);
  } else if (msib) {  // Y_(n) from the Z kept by mode n - 1's projection
    spttmc_hooi_sibling(*h->csfs[msib->csf], msib->Z.p, uptrs(h), h->J, h->Y, transposed, h->st);
    ++h->memo_hits;
  } else if (mroot) {
    const Csf& c = *h->csfs[mroot->csf];
    mroot->Z.ensure((size_t)std::max<int64_t>(1, c.nnode) * h->J[c.mid1] * round_up(h->J[c.leaf], 4));
    mroot->valid = false;
    spttmc_hooi(c, uptrs(h), h->J, h->Y, transposed, h->st, h->hooi_lo[n], h->hooi_hi[n], mroot->Z.p);
    mroot->valid = true;
  } else {
    spttmc_hooi(*h->csfs[h->hooi_csf[n]], uptrs(h), h->J, h->Y, transposed, h->st, h->hooi_lo[n], h->hooi_hi[n]);
  }
  h->Y_mode = n;
  h->Y_transposed = transposed;
  h->Y_partial = false;
  if (h->sharded) {
    if (!transposed) {
      // Y Y^T route: the ranks' rows of Y_(n) are disjoint -> allgather them
      std::vector<int64_t> off(h->hooi_bounds[n].size());
      for (size_t r = 0; r < off.size(); ++r) off[r] = h->hooi_bounds[n][r] * ld;
      dist_allgatherv_f32(h->comm, h->Yhi.p, off.data(), h->opts.world, h->st);
      dist_allgatherv_f32(h->comm, h->Ylo.p, off.data(), h->opts.world, h->st);
    } else {
      h->Y_partial = true;  // Y^T Y route: partial Gram over this rank's K range instead
    }
  }
}

// W_n = [ (X x_m U_m^T)_(n) ]_{m != n} into a kept per-(n, term set) buffer or
// h->Whi/Wlo; returns the split view.  Terms in cyclic order m = n + 1, n + 2, ...
// (the term of the factor updated last, m = n - 1, comes last: mp_sweep's overlap
// builds the others early), each term's columns padded to a multiple of 32.
// only_m >= 0: the single term m (Slice Projection, Figs. 5-6)
// mask: the terms whose columns are computed (the others are left as they are);
// fresh = false: the buffer already holds this build's other terms (never re-zeroed)
int mp_term_order(const tucker_handle* h, int n, int k) { return (n + 1 + k) % h->order; }
Split build_mp_w(tucker_handle* h, int n, int only_m = -1, uint32_t mask = ~0u, cudaStream_t s = nullptr,
                 int64_t* late_off = nullptr, bool fresh = true) {
  if (!s) s = h->st;
  // sharded: this rank's slices [mp_lo, mp_hi) of every term, columns compacted
  auto slices = [&](int m, const Csf& c, int64_t& lo, int64_t& hi) {
    lo = h->sharded ? h->mp_lo[n][m] : 0;
    hi = h->sharded ? h->mp_hi[n][m] : c.I_mid0 * c.I_mid1;
  };
  int64_t K = 0;
  for (int k = 0; k < h->order - 1; ++k) {
    const int m = mp_term_order(h, n, k);
    if (only_m >= 0 && m != only_m) continue;
    const Csf& c = *h->csfs[h->mp_csf[n][m]];
    int64_t lo, hi;
    slices(m, c, lo, hi);
    if (late_off && k == h->order - 2) *late_off = K;
    K += round_up(h->J[m] * (hi - lo), 32);
  }
  const int64_t rows = h->dims[n];
  // K-tile-major layout (Split::ktile): 32-column tiles of all rows, rows padded to 8
  const int64_t ldr = round_up(rows, 8), kpad = round_up(K, 32);
  const size_t need = (size_t)(ldr * kpad);
  auto& wk = h->wkeep[n][only_m + 1];
  const bool reuse = wk.need == need && wk.hi.p;
  if (!reuse && need > h->Whi.n) {
    size_t free_b = 0, total_b = 0;
    TK_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const double gb = 2.0 * (double)need * sizeof(float) / 1e9;
    if (2.0 * (double)need * sizeof(float) > (double)free_b + 4.0 * (double)h->Whi.n) {
      char msg[200];
      std::snprintf(msg, sizeof msg,
                    "mp_sweep: W_%d needs %.1f GB (split fp32 %lld x %lld); the fused per-slice multislice "
                    "Gram for tensors this size is not implemented",
                    n + 1, gb, (long long)rows, (long long)K);
      fail(TUCKER_E_OOM, msg);
    }
  }
  float* whi = nullptr;
  float* wlo = nullptr;
  if (reuse) {
    whi = wk.hi.p;  // same pattern: zeros still in place
    wlo = wk.lo.p;
  } else {
    size_t free_b = 0, total_b = 0;
    TK_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const size_t bytes = 2 * need * sizeof(float);
    if (!wk.hi.p && g_wkeep_bytes.load() + bytes <= total_b / 4 && bytes + total_b / 8 <= free_b) {
      wk.hi.alloc(need);
      wk.lo.alloc(need);
      wk.need = need;
      h->wkeep_bytes += bytes;
      g_wkeep_bytes += bytes;
      whi = wk.hi.p;
      wlo = wk.lo.p;
    } else {
      if (!fresh && h->Whi.n >= need) {  // the shared buffer already holds this build's other terms
        whi = h->Whi.p;
        wlo = h->Wlo.p;
        goto fill;
      }
      h->Whi.ensure(need);
      h->Wlo.ensure(need);
      whi = h->Whi.p;
      wlo = h->Wlo.p;
    }
    TK_CUDA(cudaMemsetAsync(whi, 0, need * sizeof(float), s));
    TK_CUDA(cudaMemsetAsync(wlo, 0, need * sizeof(float), s));
  }
fill:
  Split W;
  W.hi = whi;
  W.lo = wlo;
  W.rows = rows;
  W.cols = K;
  W.ld = ldr;
  W.kext = kpad;
  W.ktile = true;
  int64_t off = 0;
  for (int k = 0; k < h->order - 1; ++k) {
    const int m = mp_term_order(h, n, k);
    if (only_m >= 0 && m != only_m) continue;
    const Csf& c = *h->csfs[h->mp_csf[n][m]];
    int64_t lo, hi;
    slices(m, c, lo, hi);
    if (mask & (1u << m)) spmm_mp(c, h->U[m].p, h->J[m], W, off, s, lo, hi);
    off += round_up(h->J[m] * (hi - lo), 32);
  }
  return W;
}

// Leading eigenvectors of S (padded layout, eig_layout) -> fp64 V (d x J) in
// h->V, eigenvalues in h->theta_d (device): the persistent fused solver.
// hint: the current factor (fp32 d x J) seeds a cold slot's basis (S is I_n x I_n)
// rec: info record (sweeps: the mode, so one host sync per sweep reads them all)
void solve_eig(tucker_handle* h, int64_t d, int J, EigSlot& slot, const float* hint = nullptr,
               int rec = kMaxOrder) {
  h->V.ensure((size_t)(d * J));
  h->theta_d.ensure((size_t)J);
  h->info_d.ensure(16 * (kMaxOrder + 1));  // per record: 8 ints + 4 doubles
  h->rec_slot[rec] = &slot;
  const bool force_large = std::getenv("TUCKER_EIG_LARGE") != nullptr;  // tests
  // the direct dense solver (eig_small.cu): by default where its one-CTA form fits
  // (d <= 224, packed S in shared memory) and the iterative solver's options are at their
  // defaults (eig_max_iter / eig_tol configure the iterative solver); TUCKER_EIG_FUSED=1
  // forces the iterative solver, TUCKER_EIG_SMALL=1 the direct one up to d = 256
  // HOOI's warm-started solves converge in ~30 products at config 4 (0.5-1.2 ms per solve under
  // ncu) and stay on the fused solver; MP's and SP's (flat bulk, ~175 products, 1.4-4 ms) and the
  // cold one-off solves (HO-SVD, diagnostics) take the direct solver (~1.3 ms, gap independent)
  const bool iter_opts = h->opts.eig_max_iter > 0 || h->opts.eig_tol > 0;
  bool hooi_slot = false;
  for (int m = 0; m < kMaxOrder; ++m) hooi_slot = hooi_slot || &slot == &h->slots[0][m];
  const bool small = std::getenv("TUCKER_EIG_SMALL") != nullptr ||
                     (!std::getenv("TUCKER_EIG_FUSED") && !iter_opts && !hooi_slot &&
                      eig_direct_ws((int)std::min<int64_t>(d, 1 << 20), J) > 0);
  if (small && d <= kSmallMaxD && d >= 3 && !force_large) {
    int64_t ls = 0, rows = 0;
    eig_layout(d, &ls, &rows);
    eig_small(h->S.p, d, ls, J, h->V.p, h->theta_d.p, h->info_d.p + 16 * rec, h->eig.small, h->st);
    return;
  }
  if (d > kFusedMaxD || force_large || J > kMaxJFused) {  // config 5 MP (d = 50000), J > 112: host-driven
    int64_t ls = 0, rows = 0;
    eig_layout(d, &ls, &rows);
    eig_large(h->S.p, d, ls, J, slot, h->eig, eig_opts(h), h->V.p, h->theta_d.p, h->info_d.p + 16 * rec, h->st, hint);
    return;
  }
  eig_fused(h->S.p, d, J, slot, h->eig, eig_opts(h), h->V.p, h->theta_d.p, h->info_d.p + 16 * rec, h->st, hint);
}

// S buffer in the eigensolver's padded layout; returns its row stride
int64_t ensure_S(tucker_handle* h, int64_t d) {
  int64_t ls = 0, rows = 0;
  eig_layout(d, &ls, &rows);
  h->S.ensure((size_t)(rows * ls));
  return ls;
}

// after the stream is synchronised: fold the solver's info records [r0, r1) into
// the handle (the Lanczos / filter-bound estimates go back to each record's slot)
void eig_check(tucker_handle* h, int r0 = kMaxOrder, int r1 = kMaxOrder + 1) {
  int info[16 * (kMaxOrder + 1)];
  TK_CUDA(cudaMemcpy(info + 16 * r0, h->info_d.p + 16 * r0, 16 * (r1 - r0) * sizeof(int),
                     cudaMemcpyDeviceToHost));
  for (int r = r0; r < r1; ++r) {
    const int* in = info + 16 * r;
    if (EigSlot* sl = h->rec_slot[r]) {
      double dv[2];
      std::memcpy(dv, in + 8, sizeof(dv));
      if (dv[0] >= 0) sl->lmin = dv[0];  // a new Lanczos estimate (0: none useful)
      if (dv[1] > 0) sl->bval = dv[1];
    }
    // a broken-down or unconverged solve leaves no trustworthy basis to warm-start from
    if ((in[4] || !in[0]) && h->rec_slot[r]) h->rec_slot[r]->valid = false;
    if (in[4]) fail(TUCKER_E_CUDA, "eigensolver breakdown (non-finite Rayleigh quotient)");
    if (!in[0]) h->eig_unconverged = true;
    h->eig.stat_outer += in[1];
    h->eig.stat_matvec += in[2];
    h->eig.stat_sweeps += in[3];
  }
}

// timing events of one sweep (recorded on the handle stream, read after its one sync)
struct SweepEvents {
  std::vector<cudaEvent_t> e;
  explicit SweepEvents(int n) : e((size_t)n, nullptr) {
    for (auto& x : e) TK_CUDA(cudaEventCreate(&x));
  }
  ~SweepEvents() {
    for (auto x : e)
      if (x) cudaEventDestroy(x);
  }
  SweepEvents(const SweepEvents&) = delete;
  SweepEvents& operator=(const SweepEvents&) = delete;
  float ms(int i, int j) const {
    float t = 0;
    TK_CUDA(cudaEventElapsedTime(&t, e[i], e[j]));
    return t;
  }
};

void factor_from_S(tucker_handle* h, int n, const Split& A, bool transposed, EigSlot& slot, bool partial_gram);

// MP's multislice Gram without the dense W (order 3, tensors whose W_n would not fit):
// h->S = sum over the terms m != n (only_m >= 0: that term) of sum_s P_s P_s^T, built
// slice by slice from the orderings (root o, mid n, leaf m) (mp_sparse.cu); sharded:
// this rank's slices, summed by an fp64 allreduce.  Returns the d x 0 Split view the
// factor step needs (rows = I_n).
bool mp_use_sparse(tucker_handle* h, int n, int only_m) {
  if (h->order != 3) return false;
  if (const char* e = std::getenv("TUCKER_MP_SPARSE")) return std::atoi(e) != 0;  // tests / experiments
  int64_t K = 0;
  for (int m = 0; m < h->order; ++m) {
    if (m == n || (only_m >= 0 && m != only_m)) continue;
    const Csf& c = *h->csfs[h->mp_csf[n][m]];
    K += h->J[m] * c.I_mid0;
  }
  size_t free_b = 0, total_b = 0;
  TK_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const double wbytes = 8.0 * (double)round_up(h->dims[n], 8) * (double)round_up(K, 32);
  return wbytes > 0.4 * (double)free_b;
}

Split build_mp_gram_sparse(tucker_handle* h, int n, int only_m) {
  const int64_t d = h->dims[n];
  const int64_t lds = ensure_S(h, d);
  int64_t ls = 0, rows = 0;
  eig_layout(d, &ls, &rows);
  TK_CUDA(cudaMemsetAsync(h->S.p, 0, (size_t)(rows * ls) * sizeof(double), h->st));
  size_t free_b = 0, total_b = 0;
  TK_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const size_t max_p = std::max<size_t>((size_t)1 << 24, std::min<size_t>(free_b / 3, (size_t)16 << 30) / sizeof(float));
  for (int m = 0; m < h->order; ++m) {
    if (m == n || (only_m >= 0 && m != only_m)) continue;
    const int o = 3 - n - m;
    const Csf& c = *h->csfs[h->mp_csf[o][m]];  // root o (the slice), mid n, leaf m
    const int64_t lo = h->sharded ? h->mp_lo[n][m] : 0, hi = h->sharded ? h->mp_hi[n][m] : c.I_root;
    mp_sparse_term(c, h->U[m].p, h->J[m], lo, hi, h->S.p, lds, h->Pmp, max_p, h->st);
  }
  mp_sparse_mirror(h->S.p, d, lds, h->st);
  Split A;
  A.rows = d;
  return A;
}

// U_n from the eigenvectors of the Gram of the split matrix A (= Y, Y^T or W)
// Sharded: a partial Gram (MP: this rank's W columns; HOOI Y^T Y route: this
// rank's K range of Y^T, rounded out to 32 columns -- the other ranks' columns
// in the rounding are zero here) summed by an fp64 allreduce.
// ev_gram (nullable) is recorded after the Gram; the solver writes info record n
// (no host synchronisation here: the sweep reads its records once, at its end)
void update_factor(tucker_handle* h, int n, const Split& A, bool transposed, EigSlot& slot, cudaEvent_t ev_gram,
                   bool partial_gram) {
  const int64_t d = A.rows;
  const int J = (int)h->J[n];
  const int64_t lds = ensure_S(h, d);
  if (partial_gram && transposed) {
    const int64_t lo = h->hooi_lo[n], hi = h->hooi_hi[n];
    const int64_t k0 = std::min(A.ld, lo / 32 * 32), k1 = std::min(A.ld, round_up(std::max(hi, lo), 32));
    Split Ar = A;
    Ar.hi = A.hi + k0;
    Ar.lo = A.lo + k0;
    Ar.kext = k1 - k0;
    if (Ar.kext == 0) Ar.ld = 0;  // empty shard: gram_syrk writes S = 0
    gram_syrk(Ar, h->S.p, lds, h->gram, h->st);
  } else {
    gram_syrk(A, h->S.p, lds, h->gram, h->st);
  }
  if (partial_gram) dist_allreduce_f64(h->comm, h->S.p, d * lds, h->st);
  if (ev_gram) TK_CUDA(cudaEventRecord(ev_gram, h->st));
  factor_from_S(h, n, A, transposed, slot, partial_gram);
}

// U_n from the Gram already in h->S (I_n x I_n, or prod J x prod J on the Y^T Y route)
void factor_from_S(tucker_handle* h, int n, const Split& A, bool transposed, EigSlot& slot, bool partial_gram) {
  const int64_t d = A.rows;
  const int J = (int)h->J[n];
  memo_invalidate(h, n);
  solve_eig(h, d, J, slot, transposed ? nullptr : h->U[n].p, n);
  if (!transposed) {
    canon_to_f32(h->V.p, J, d, J, h->U[n].p, h->st);
  } else {
    // Y^T Y route: U = Y_(n) V Theta^{-1/2} = (Y^T)^T V Theta^{-1/2}, then CholQR2
    TK_LAUNCH(k_scale_cols_rsqrt, gridn(d * J), 256, 0, h->st, h->V.p, d, J, h->theta_d.p);
    const int64_t I = h->dims[n];
    h->Ufull.ensure((size_t)(I * J));
    MatRef a;
    a.t = Elt::SPLIT; a.p = A.hi; a.lo = A.lo; a.ld = A.ld; a.trans = true;
    MatRef b;
    b.t = Elt::F64; b.p = h->V.p; b.ld = J; b.trans = false;
    dgemm(I, J, d, 1.0, a, b, 0.0, h->Ufull.p, J, 0.0, nullptr, 0, h->eig.dense, h->st);
    // sharded: this rank computed the rows of its shard (the others are zero: Y was) -> allgather
    if (partial_gram) {
      std::vector<int64_t> off(h->hooi_bounds[n].size());
      for (size_t r = 0; r < off.size(); ++r) off[r] = h->hooi_bounds[n][r] * J;
      dist_allgatherv_f64(h->comm, h->Ufull.p, off.data(), h->opts.world, h->st);
    }
    cholqr2(h->Ufull.p, J, I, J, h->eig, h->st);
    canon_to_f32(h->Ufull.p, J, I, J, h->U[n].p, h->st);
  }
}

// One MP / SP factor update of mode n (only_m >= 0: the single term of Slice
// Projection): the dense-W route (SpMM + Gram) or, when W_n would not fit, the sparse
// multislice Gram; ev_proj / ev_gram are recorded after the W build / the Gram.
void mp_update(tucker_handle* h, int n, int only_m, EigSlot& slot, cudaEvent_t ev_proj, cudaEvent_t ev_gram) {
  if (mp_use_sparse(h, n, only_m)) {
    TK_CUDA(cudaEventRecord(ev_proj, h->st));
    Split A = build_mp_gram_sparse(h, n, only_m);
    if (h->sharded) {
      int64_t ls = 0, rows = 0;
      eig_layout(A.rows, &ls, &rows);
      dist_allreduce_f64(h->comm, h->S.p, A.rows * ls, h->st);
    }
    TK_CUDA(cudaEventRecord(ev_gram, h->st));
    factor_from_S(h, n, A, false, slot, h->sharded);
    return;
  }
  Split W = only_m >= 0 ? build_mp_w(h, n, only_m) : build_mp_w(h, n);
  TK_CUDA(cudaEventRecord(ev_proj, h->st));
  update_factor(h, n, W, false, slot, ev_gram, h->sharded);
}

// MP overlap (mp_sweep): M_n = sum_{m != n} W_m W_m^T, and only the term of the factor
// updated last (m = n - 1) depends on the eigensolve just before; the other terms' W columns
// and their partial Gram are built on a second stream while that eigensolve runs (one CTA
// for MP's d <= 224 direct solver, the fused solver's few CTAs otherwise).  Same arithmetic
// as mp_update; the Gram sum is split into S2 (early terms) + the late term, in fp64.
// Dense-W route, unsharded, order >= 3; TUCKER_MP_OVERLAP=0 disables it.
bool mp_overlap_ok(tucker_handle* h, int n) {
  const char* e = std::getenv("TUCKER_MP_OVERLAP");
  const bool off = e && e[0] == '0';
  return !off && !h->sharded && h->order >= 3 && !mp_use_sparse(h, n, -1);
}
// mode n's MP eigensolve is the one-CTA direct solver (solve_eig's rule): only then is there a
// GPU to share -- the fused solver is a cooperative grid over every SM (config 2's d = 1000)
bool mp_eig_direct(tucker_handle* h, int n) {
  const int64_t d = h->dims[n];
  const bool iter_opts = h->opts.eig_max_iter > 0 || h->opts.eig_tol > 0;
  return !std::getenv("TUCKER_EIG_FUSED") && !iter_opts && d >= 3 && d <= kSmallMaxD &&
         eig_direct_ws((int)d, (int)h->J[n]) > 0;
}



// the early terms of mode n (all but m = n - 1) into W_n and S2, on h->st2
static bool mp_timeline() {
  const char* e = std::getenv("TUCKER_MP_TIMELINE");
  return e && e[0] == '1';
}
void mp_side(tucker_handle* h, int n, cudaEvent_t* tl = nullptr) {
  const int N = h->order, late = (n + N - 1) % N;
  uint32_t mask = 0;
  for (int m = 0; m < N; ++m)
    if (m != n && m != late) mask |= 1u << m;
  const AllocScope as(h->st2);
  // the eigensolve holds one SM: persistent side kernels size their grids to the others
  // (a grid that needs the held SM's slots runs its last blocks after a whole block's share)
  const SmReserveScope rs(1);
  int64_t off_late = 0;
  Split W = build_mp_w(h, n, -1, mask, h->st2, &off_late);
  if (tl) TK_CUDA(cudaEventRecord(tl[2], h->st2));
  Split We = W;
  We.kext = off_late;
  We.cols = off_late;
  int64_t ls = 0, rows = 0;  // S2 in S's padded layout (h->S itself is in use by the eigensolve)
  eig_layout(W.rows, &ls, &rows);
  h->S2.ensure((size_t)(rows * ls));
  gram_syrk(We, h->S2.p, ls, h->gram2, h->st2, nullptr, 0.5 * (double)W.rows * (W.rows + 1) * (double)W.K());
  if (tl) TK_CUDA(cudaEventRecord(tl[3], h->st2));
  h->side_ready[n] = true;
}

void mp_update_overlap(tucker_handle* h, int n, EigSlot& slot, cudaEvent_t ev_proj, cudaEvent_t ev_gram, int next) {
  if (!h->st2) {
    // the eigensolve's CTA(s) must be dispatched before the side kernels fill every SM (the SpMM
    // blocks are persistent): it runs on a greatest-priority stream, the side work on a least one
    int least = 0, greatest = 0;
    TK_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    TK_CUDA(cudaStreamCreateWithPriority(&h->st2, cudaStreamNonBlocking, least));
    TK_CUDA(cudaStreamCreateWithPriority(&h->st_hi, cudaStreamNonBlocking, greatest));
    TK_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    TK_CUDA(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
    TK_CUDA(cudaEventCreateWithFlags(&h->ev_eig, cudaEventDisableTiming));
  }
  const int N = h->order, late = (n + N - 1) % N;
  const int64_t d = h->dims[n];
  const int64_t lds = ensure_S(h, d);
  cudaEvent_t* tl = h->tl[n];  // always on: seven event records per mode
  for (int q = 0; q < 8; ++q)
    if (!tl[q]) TK_CUDA(cudaEventCreate(&tl[q]));
  h->tl_rec[n] = 0;
  if (h->side_ready[n]) {  // early terms done on st2: the late term, S = S2 + W_late W_late^T
    TK_CUDA(cudaStreamWaitEvent(h->st, h->ev_join, 0));
    if (tl) TK_CUDA(cudaEventRecord(tl[4], h->st));
    int64_t off_late = 0;
    Split W = build_mp_w(h, n, -1, 1u << late, h->st, &off_late, false);
    TK_CUDA(cudaEventRecord(ev_proj, h->st));
    if (tl) TK_CUDA(cudaEventRecord(tl[5], h->st));
    Split Wl = W;
    const int64_t sh = off_late / 32 * 32 * W.ld;  // K-tile-major: whole 32-column tiles
    Wl.hi = W.hi + sh;
    Wl.lo = W.lo + sh;
    Wl.kext = W.kext - off_late;
    Wl.cols = W.cols - off_late;
    gram_syrk(Wl, h->S.p, lds, h->gram, h->st, h->S2.p, 0.5 * (double)W.rows * (W.rows + 1) * (double)W.K());
    if (tl) TK_CUDA(cudaEventRecord(tl[6], h->st));
    h->side_ready[n] = false;
    h->tl_rec[n] |= 4u;
  } else {
    TK_CUDA(cudaEventRecord(tl[4], h->st));
    Split W = build_mp_w(h, n);
    TK_CUDA(cudaEventRecord(ev_proj, h->st));
    TK_CUDA(cudaEventRecord(tl[5], h->st));
    gram_syrk(W, h->S.p, lds, h->gram, h->st);
    TK_CUDA(cudaEventRecord(tl[6], h->st));
    h->tl_rec[n] |= 8u;  // whole build: N - 1 terms
  }
  TK_CUDA(cudaEventRecord(ev_gram, h->st));
  TK_CUDA(cudaEventRecord(h->ev_fork, h->st));
  if (tl) TK_CUDA(cudaEventRecord(tl[0], h->st));
  {  // the eigensolve (and the factor update) on the greatest-priority stream, launched first
    TK_CUDA(cudaStreamWaitEvent(h->st_hi, h->ev_fork, 0));
    cudaStream_t main_st = h->st;
    h->st = h->st_hi;
    TK_CUDA(cudaEventRecord(tl[7], h->st_hi));  // (re-recorded right after the direct solver's kernel)
    g_eig_kernel_event = tl[7];
    try {
      const AllocScope as(h->st_hi);
      Split A;
      A.rows = d;
      factor_from_S(h, n, A, false, slot, false);
    } catch (...) {
      g_eig_kernel_event = nullptr;
      h->st = main_st;
      throw;
    }
    g_eig_kernel_event = nullptr;
    h->st = main_st;
    TK_CUDA(cudaEventRecord(h->ev_eig, h->st_hi));
    if (tl) TK_CUDA(cudaEventRecord(tl[1], h->st_hi));
    h->tl_rec[n] |= 1u;
  }
  if (next >= 0) {  // every factor but U_n is final: the next mode's early terms meanwhile
    TK_CUDA(cudaStreamWaitEvent(h->st2, h->ev_fork, 0));
    mp_side(h, next, tl);
    TK_CUDA(cudaEventRecord(h->ev_join, h->st2));
    h->tl_rec[n] |= 2u;
  }
  TK_CUDA(cudaStreamWaitEvent(h->st, h->ev_eig, 0));
}

// G_(N) = U_N^T Y_(N) from h->Y (must be the projection of the last mode with
// the current factors), then ||G||^2 and the fit.
double core_from_y(tucker_handle* h) {
  const int n = h->order - 1;
  const int64_t P = prod_J_except(h, n);
  const int64_t JN = h->J[n];
  const int64_t I = h->dims[n];
  h->G64.ensure((size_t)(JN * P));
  MatRef a;
  a.t = Elt::F32; a.p = h->U[n].p; a.ld = JN; a.trans = true;
  MatRef b;
  b.t = Elt::SPLIT; b.p = h->Y.hi; b.lo = h->Y.lo; b.ld = h->Y.ld; b.trans = h->Y_transposed;
  dgemm(JN, P, I, 1.0, a, b, 0.0, h->G64.p, P, 0.0, nullptr, 0, h->eig.dense, h->st);
  if (h->Y_partial) dist_allreduce_f64(h->comm, h->G64.p, JN * P, h->st);  // partial sums over the row shards
  h->scal.ensure(2);
  TK_LAUNCH(k_core_fit, 1, 512, 0, h->st, h->G64.p, JN * P, h->normX2, h->scal.p);
  double out[2];
  TK_CUDA(cudaMemcpyAsync(out, h->scal.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  TK_CUDA(cudaStreamSynchronize(h->st));
  h->G_valid = true;
  h->last_g2 = out[0];
  return out[1];
}

double compute_core(tucker_handle* h) {
  const int n = h->order - 1;
  const bool tr = prod_J_except(h, n) < h->dims[n] && h->J[n] <= kMaxBlock;
  project_hooi(h, n, tr);
  return core_from_y(h);
}

template <typename T>
std::vector<T> to_host(const DBuf<T>& b, int64_t n, cudaStream_t st) {
  std::vector<T> v((size_t)n);
  if (n > 0) TK_CUDA(cudaMemcpyAsync(v.data(), b.p, n * sizeof(T), cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  return v;
}

// Work-balanced contiguous shards: HOOI mode n by root slice of
// its CSF (work J_leaf nnz + prod_{q != n} J_q fibers per slice, the SpTTMc flop
// model; order 4: J_leaf nnz), MP term (n, m) by slice = mid index (work J_m
// (nnz + fibers) per slice: the leaf SpMM and its W writes).
void make_shards(tucker_handle* h) {
  const int W = h->opts.world, r = h->opts.rank;
  std::vector<int64_t> b((size_t)W + 1);
  for (int n = 0; n < h->order; ++n) {
    const Csf& c = *h->csfs[h->hooi_csf[n]];
    const auto sp = to_host(c.slice_ptr, c.I_root + 1, h->st);
    const auto fp = to_host(c.fib_ptr, c.nfib + 1, h->st);
    std::vector<int32_t> np;
    if (c.order == 4) np = to_host(c.node_ptr, c.nnode + 1, h->st);
    const double P = (double)prod_J_except(h, n), Jl = (double)h->J[c.leaf];
    std::vector<double> w((size_t)c.I_root);
    for (int64_t i = 0; i < c.I_root; ++i) {
      if (c.order == 3) {
        w[i] = Jl * (double)(fp[sp[i + 1]] - fp[sp[i]]) + P * (double)(sp[i + 1] - sp[i]);
      } else {
        w[i] = Jl * (double)(fp[np[sp[i + 1]]] - fp[np[sp[i]]]);
      }
    }
    shard_bounds(w.data(), c.I_root, W, b.data());
    h->hooi_lo[n] = b[r];
    h->hooi_hi[n] = b[r + 1];
    h->hooi_bounds[n] = b;
    for (int m = 0; m < h->order; ++m) {
      if (m == n) continue;
      const Csf& t = *h->csfs[h->mp_csf[n][m]];
      const int64_t ns = t.I_mid0 * t.I_mid1;
      const auto tf = to_host(t.fib_ptr, t.nfib + 1, h->st);
      const auto m0 = to_host(t.fib_mid0, t.nfib, h->st);
      std::vector<int32_t> m1;
      if (t.mid1 >= 0) m1 = to_host(t.fib_mid1, t.nfib, h->st);
      std::vector<double> ws((size_t)ns, 0.0);
      for (int64_t f = 0; f < t.nfib; ++f) {
        const int64_t mk = t.mid1 >= 0 ? (int64_t)m0[f] * t.I_mid1 + m1[f] : m0[f];
        ws[mk] += (double)h->J[m] * (double)(tf[f + 1] - tf[f] + 1);
      }
      shard_bounds(ws.data(), ns, W, b.data());
      h->mp_lo[n][m] = b[r];
      h->mp_hi[n][m] = b[r + 1];
    }
  }
}

// The paper's stop rule (Eq. 10; MP: Appendix): sweep until
// Delta_fit(t) = fit(t) - fit(t-1) < tol (fit(0) = 0) or max_sweeps sweeps,
// from the factors currently in the handle.  fits[t] per sweep (length
// max_sweeps, nullable); *sweeps_done = t.  An unconverged eigensolve is not
// fatal here (reported as TUCKER_E_CONVERGE after the loop, like the sweeps).
template <typename SweepFn>
int run_until(tucker_handle* h, int max_sweeps, double tol, double* fits, int* sweeps_done, SweepFn sweep) {
  if (!h || max_sweeps < 1 || !(tol >= 0)) return TUCKER_E_ARG;
  double old = 0.0;
  int t = 0, rc_all = TUCKER_OK;
  while (t < max_sweeps) {
    double fit = 0.0;
    const int rc = sweep(h, &fit);
    if (rc == TUCKER_E_CONVERGE) rc_all = rc;
    else if (rc != TUCKER_OK) return rc;
    if (fits) fits[t] = fit;
    ++t;
    if (fit - old < tol) break;
    old = fit;
  }
  if (sweeps_done) *sweeps_done = t;
  return rc_all;
}

int validate_factor(const float* U, int64_t I, int64_t J) {
  // max |U^T U - I| <= 1e-5 (host check on the caller's copy)
  std::vector<double> G((size_t)(J * J), 0.0);
  for (int64_t i = 0; i < I; ++i)
    for (int64_t a = 0; a < J; ++a) {
      const double ua = U[i * J + a];
      if (!std::isfinite(ua)) return TUCKER_E_FACTOR;
      for (int64_t b = a; b < J; ++b) G[a * J + b] += ua * (double)U[i * J + b];
    }
  for (int64_t a = 0; a < J; ++a)
    for (int64_t b = a; b < J; ++b)
      if (std::fabs(G[a * J + b] - (a == b ? 1.0 : 0.0)) > 1e-5) return TUCKER_E_FACTOR;
  return TUCKER_OK;
}

}  // namespace

extern "C" {

void tucker_default_opts(tucker_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->device = 0;
  o->rank = 0;
  o->world = 1;
}

const char* tucker_strerror(int code) {
  switch (code) {
    case TUCKER_OK: return "ok";
    case TUCKER_E_ARG: return "invalid argument";
    case TUCKER_E_INDEX: return "index out of range";
    case TUCKER_E_DUP: return "duplicate coordinate";
    case TUCKER_E_VALUE: return "non-finite value or zero tensor";
    case TUCKER_E_FACTOR: return "initial factor not orthonormal";
    case TUCKER_E_CUDA: return "CUDA error";
    case TUCKER_E_NCCL: return "NCCL error";
    case TUCKER_E_OOM: return "out of device memory";
    case TUCKER_E_STATE: return "call out of order";
    case TUCKER_E_CONVERGE: return "eigensolver did not reach tolerance";
    default: return "unknown error";
  }
}

const char* tucker_last_error(const tucker_handle* h) { return h ? h->last_error.c_str() : ""; }

static int sm_count(int dev) {
  int n = 0;
  TK_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}

int tucker_init(tucker_handle** out, int order, const int64_t* dims, const int64_t* core,
                int64_t nnz, const int32_t* const* idx, const float* vals, const float* const* U0,
                const tucker_opts* opts) {
  if (!out || !dims || !core || !idx || !vals || !U0) return TUCKER_E_ARG;
  *out = nullptr;
  if (order < 2 || order > kMaxOrder || nnz <= 0 || nnz >= (int64_t)1 << 31) return TUCKER_E_ARG;
  tucker_opts o;
  tucker_default_opts(&o);
  if (opts) o = *opts;
  if (o.world < 1 || o.rank < 0 || o.rank >= o.world) return TUCKER_E_ARG;
  const bool host_coll = (o.flags & TUCKER_HOST_COLLECTIVES) != 0;
  if (o.world > 1 && !o.nccl_unique_id && !host_coll) return TUCKER_E_ARG;
  uint64_t cells = 1;  // the CSF sort keys pack every coordinate into one 64-bit key
  for (int n = 0; n < order; ++n) {
    if (dims[n] < 1 || dims[n] >= (int64_t)1 << 31) return TUCKER_E_ARG;
    if (core[n] < 1 || core[n] > dims[n] || core[n] > kMaxJ) return TUCKER_E_ARG;
    if (!idx[n] || !U0[n]) return TUCKER_E_ARG;
    if (__builtin_mul_overflow(cells, (uint64_t)dims[n], &cells)) return TUCKER_E_ARG;
  }
  // J_n <= prod_{q != n} J_q: Y_(n) has rank <= prod_{q != n} J_q, so a larger J_n
  // has no J_n-dimensional dominant subspace to return (S:136 rank deficiency)
  for (int n = 0; n < order; ++n) {
    int64_t P = 1;
    for (int q = 0; q < order; ++q)
      if (q != n) P *= core[q];
    if (core[n] > P) return TUCKER_E_ARG;
  }
  const bool on_dev = (o.flags & TUCKER_INPUT_ON_DEVICE) != 0;
  if (!on_dev)
    for (int n = 0; n < order; ++n) {
      const int rc = validate_factor(U0[n], dims[n], core[n]);
      if (rc) return rc;
    }
  // orders 2 and 5..8 (HOOI only, gen.cu): one rank (the sharded sweep is built on the CSF)
  const bool generic = order != 3 && order != 4;
  if (generic && o.world > 1) return TUCKER_E_ARG;
  auto h = std::make_unique<tucker_handle>();
  h->order = order;
  h->generic = generic;
  h->opts = o;
  for (int n = 0; n < order; ++n) {
    h->dims[n] = dims[n];
    h->J[n] = core[n];
  }
  for (auto& r : h->mp_csf)
    for (int& v : r) v = -1;
  const int rc = guarded(h.get(), [&]() -> int {
    if (o.stream) {
      h->st = (cudaStream_t)o.stream;
    } else {
      TK_CUDA(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
      h->own_stream = true;
    }
    mempool_retain(o.device);
    g_alloc_stream = h->st;  // the scope (guarded) restores the previous value
    // TUCKER_PROFILE_INIT=1: phase times on stderr (host clock, stream synchronised)
    const bool prof = std::getenv("TUCKER_PROFILE_INIT") != nullptr;
    auto tp = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
      if (!prof) return;
      TK_CUDA(cudaStreamSynchronize(h->st));
      const auto now = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[init] %-28s %8.3f ms\n", what,
                   std::chrono::duration<double, std::milli>(now - tp).count());
      tp = now;
    };
    const cudaMemcpyKind kind = on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    Coo& c = h->coo;
    c.order = order;
    c.nnz = nnz;
    for (int n = 0; n < order; ++n) {
      c.dims[n] = dims[n];
      c.idx[n].alloc(nnz);
      TK_CUDA(cudaMemcpyAsync(c.idx[n].p, idx[n], nnz * sizeof(int32_t), kind, h->st));
      h->U[n].alloc((size_t)(dims[n] * core[n]));
      TK_CUDA(cudaMemcpyAsync(h->U[n].p, U0[n], dims[n] * core[n] * sizeof(float), kind, h->st));
    }
    c.val.alloc(nnz);
    TK_CUDA(cudaMemcpyAsync(c.val.p, vals, nnz * sizeof(float), kind, h->st));
    mark("H2D copies + allocs");
    if (h->generic) {  // orders 2, 5..8: sorted COO per mode (gen.cu), HOOI only
      gen_build(c, h->gen, h->st);
      h->normX2 = coo_norm2(c, h->st);
      if (!(h->normX2 > 0) || !std::isfinite(h->normX2))
        fail(TUCKER_E_VALUE, "tucker_init: ||X|| = 0 or not finite");
      for (int n = 0; n < order; ++n) c.idx[n].release();
      c.val.release();
      TK_CUDA(cudaStreamSynchronize(h->st));
      return TUCKER_OK;
    }
    coo_validate_compact(c, h->st);
    mark("validate");
    h->normX2 = coo_norm2(c, h->st);
    mark("norm");
    if (!(h->normX2 > 0) || !std::isfinite(h->normX2))
      fail(TUCKER_E_VALUE, "tucker_init: ||X|| = 0 or not finite");
    // orderings: root n, leaf m, mids = the other modes ascending
    for (int n = 0; n < order; ++n) {
      for (int m = 0; m < order; ++m) {
        if (m == n) continue;
        int mids[2] = {-1, -1}, nm = 0;
        for (int q = 0; q < order; ++q)
          if (q != n && q != m) mids[nm++] = q;
        auto cs = std::make_unique<Csf>();
        csf_build(c, *cs, n, mids[0], order == 4 ? mids[1] : -1, m, h->st);
        mark("csf_build");
        h->mp_csf[n][m] = (int)h->csfs.size();
        h->csfs.push_back(std::move(cs));
      }
      // HOOI leaf: minimise the SpTTMc flop model
      // J_leaf * nnz (fiber stage) + (prod_{q != n} J_q) * nfib (Kronecker
      // stage) over the built orderings (ties: highest mode id)
      int best = -1;
      double best_cost = 0;
      double Pn = 1;
      for (int q = 0; q < order; ++q)
        if (q != n) Pn *= (double)h->J[q];
      for (int m = 0; m < order; ++m) {
        if (m == n) continue;
        const Csf& cm = *h->csfs[h->mp_csf[n][m]];
        const double cost = (double)h->J[m] * (double)cm.nnz + Pn * (double)(order == 4 ? cm.nnode : cm.nfib);
        if (best < 0 || cost <= best_cost) {
          best = m;
          best_cost = cost;
        }
      }
      h->hooi_csf[n] = h->mp_csf[n][best];
    }
    if (o.nccl_unique_id || host_coll) {
      h->comm = o.nccl_unique_id ? dist_comm_init(o.nccl_unique_id, o.world, o.rank) : dist_comm_host();
      h->sharded = true;
      make_shards(h.get());
    }
    // HOOI partial-contraction reuse (order 4, one rank; TUCKER_HOOI_MEMO=0 disables): modes
    // (0, 1) share Z = X x_2 U_2^T x_3 U_3^T, modes (2, 3) share Z = X x_0 U_0^T x_1 U_1^T.
    // Mode p takes the ordering (p; p + 1; x; y) with the cheaper leaf; (2; 3; x; y) is an extra
    // ordering (the MP orderings keep their mids ascending).  Only where the GEMM-form kernel
    // (the one that keeps Z) runs by default and Z fits an eighth of the free memory.
    {
      const char* me = std::getenv("TUCKER_HOOI_MEMO");
      const bool want = order == 4 && !h->sharded && !(me && me[0] == '0');
      for (int pr = 0; want && pr < 2; ++pr) {
        const int p = 2 * pr, q = p + 1, x = pr == 0 ? 2 : 0, y = pr == 0 ? 3 : 1;
        // leaf: the smaller J (ties: the higher mode), as in the HOOI flop model (nnode is the same)
        const int leaf = h->J[x] < h->J[y] ? x : y, mid1 = leaf == x ? y : x;
        int ci = -1;
        if (pr == 0) {
          ci = h->mp_csf[p][leaf];  // mids ascending = (1, mid1)
        } else {
          auto cs = std::make_unique<Csf>();
          csf_build(c, *cs, p, q, mid1, leaf, h->st);
          mark("csf_build (memo)");
          ci = (int)h->csfs.size();
          h->csfs.push_back(std::move(cs));
        }
        const Csf& cm = *h->csfs[ci];
        size_t fr = 0, tot = 0;
        TK_CUDA(cudaMemGetInfo(&fr, &tot));
        const double zbytes = 4.0 * (double)cm.nnode * (double)h->J[mid1] * (double)round_up(h->J[leaf], 4);
        if (cm.mid0 != q || !spttmc4g_fma_default(cm, h->J) || zbytes > (double)fr / 8) {
          if (pr == 1) h->csfs.pop_back();
          continue;
        }
        h->memo[pr].csf = ci;
        h->memo[pr].root = p;
        h->memo[pr].sib = q;
        h->hooi_csf[p] = ci;
      }
    }
    for (int n = 0; n < order; ++n) {  // order 4: Jm = J_mid0 J_mid1 (the partial row is prod_{q != n} J_q)
      Csf& ch = *h->csfs[h->hooi_csf[n]];
      const int64_t Jm = h->J[ch.mid0] * (order == 4 ? h->J[ch.mid1] : 1);
      spttmc_plan(ch, Jm, h->J[ch.leaf], sm_count(h->opts.device), h->st, h->hooi_lo[n], h->hooi_hi[n]);
    }
    mark("spttmc plans");
    // the COO copy is no longer needed
    for (int n = 0; n < order; ++n) c.idx[n].release();
    c.val.release();
    TK_CUDA(cudaStreamSynchronize(h->st));
    return TUCKER_OK;
  });
  if (rc != TUCKER_OK) {
    // keep the message for the caller through stderr (no handle is returned)
    std::fprintf(stderr, "tucker_init: %s\n", h->last_error.c_str());
    // free the handle's buffers (stream-ordered on h->st) before the stream goes
    const bool own = h->own_stream;
    cudaStream_t st = h->st;
    if (h->comm) dist_comm_destroy(h->comm);
    h.reset();
    if (own && st) cudaStreamDestroy(st);
    return rc;
  }
  *out = h.release();
  return TUCKER_OK;
}

int tucker_set_factors(tucker_handle* h, const float* const* U) {
  if (!h || !U) return TUCKER_E_ARG;
  const bool on_dev = (h->opts.flags & TUCKER_INPUT_ON_DEVICE) != 0;
  for (int n = 0; n < h->order; ++n) {
    if (!U[n]) return TUCKER_E_ARG;
    if (!on_dev) {
      const int rc = validate_factor(U[n], h->dims[n], h->J[n]);
      if (rc) return rc;
    }
  }
  return guarded(h, [&]() -> int {
    for (int n = 0; n < h->order; ++n)
      TK_CUDA(cudaMemcpyAsync(h->U[n].p, U[n], h->dims[n] * h->J[n] * sizeof(float),
                              on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->st));
    TK_CUDA(cudaStreamSynchronize(h->st));
    h->G_valid = false;
    memo_invalidate(h, -1);
    for (auto& row : h->slots)
      for (auto& s : row) s.valid = false;
    return TUCKER_OK;
  });
}

int hooi_sweep(tucker_handle* h, int sweeps, double* fit_per_sweep, float* stage_ms) {
  if (!h || sweeps < 1) return TUCKER_E_ARG;
  return guarded(h, [&]() -> int {
    h->eig_unconverged = false;
    const int N = h->order;
    // events per mode: [4n] start, [4n+1] projected, [4n+2] Gram, [4n+3] factor; [4N], [4N+1] core
    SweepEvents ev(4 * N + 2);
    for (int s = 0; s < sweeps; ++s) {
      for (int n = 0; n < N; ++n) {
        // Y^T Y is the smaller Gram; its back-transform's CholQR2 handles J_n <= kMaxBlock
        const bool tr = prod_J_except(h, n) < h->dims[n] && h->J[n] <= kMaxBlock;
        TK_CUDA(cudaEventRecord(ev.e[4 * n], h->st));
        project_hooi(h, n, tr);
        TK_CUDA(cudaEventRecord(ev.e[4 * n + 1], h->st));
        update_factor(h, n, h->Y, tr, h->slots[0][n], ev.e[4 * n + 2], h->sharded && tr);
        TK_CUDA(cudaEventRecord(ev.e[4 * n + 3], h->st));
      }
      // G_(N) = U_N^T Y_(N) is free after the last mode (Fig. 4); reading
      // the fit is the sweep's one host synchronisation
      TK_CUDA(cudaEventRecord(ev.e[4 * N], h->st));
      const double fit = core_from_y(h);
      TK_CUDA(cudaEventRecord(ev.e[4 * N + 1], h->st));
      TK_CUDA(cudaEventSynchronize(ev.e[4 * N + 1]));
      eig_check(h, 0, N);
      float ms[4] = {0, 0, 0, ev.ms(4 * N, 4 * N + 1)};
      for (int n = 0; n < N; ++n) {
        ms[0] += ev.ms(4 * n, 4 * n + 1);
        ms[1] += ev.ms(4 * n + 1, 4 * n + 2);
        ms[2] += ev.ms(4 * n + 2, 4 * n + 3);
      }
      if (fit_per_sweep) fit_per_sweep[s] = fit;
      if (stage_ms)
        for (int q = 0; q < 4; ++q) stage_ms[4 * s + q] = ms[q];
    }
    return h->eig_unconverged ? TUCKER_E_CONVERGE : TUCKER_OK;
  });
}

int mp_sweep(tucker_handle* h, int sweeps, double* fit_per_sweep, float* stage_ms) {
  if (!h || sweeps < 1 || h->generic) return TUCKER_E_ARG;  // MP: orders 3, 4 (reading A18)
  return guarded(h, [&]() -> int {
    for (auto& r : h->side_ready) r = false;
    if (h->st2) TK_CUDA(cudaStreamSynchronize(h->st2));  // nothing of an earlier call still in flight
    h->eig_unconverged = false;
    h->G_valid = false;
    const int N = h->order;
    SweepEvents ev(4 * N + 2);
    for (int s = 0; s < sweeps; ++s) {
      for (int n = 0; n < N; ++n) {
        TK_CUDA(cudaEventRecord(ev.e[4 * n], h->st));
        const int nn = (n + 1) % N;
        const bool more = n + 1 < N || s + 1 < sweeps;
        if (mp_overlap_ok(h, n)) {
          mp_update_overlap(h, n, h->slots[1][n], ev.e[4 * n + 1], ev.e[4 * n + 2],
                            more && mp_overlap_ok(h, nn) && mp_eig_direct(h, n) ? nn : -1);
        } else {
          mp_update(h, n, -1, h->slots[1][n], ev.e[4 * n + 1], ev.e[4 * n + 2]);
        }
        TK_CUDA(cudaEventRecord(ev.e[4 * n + 3], h->st));
      }
      h->G_valid = false;
      TK_CUDA(cudaEventRecord(ev.e[4 * N], h->st));
      if (fit_per_sweep) fit_per_sweep[s] = compute_core(h);
      TK_CUDA(cudaEventRecord(ev.e[4 * N + 1], h->st));
      TK_CUDA(cudaEventSynchronize(ev.e[4 * N + 1]));  // the sweep's one host synchronisation
      for (int n = 0; n < N; ++n) {  // overlap accounting (events of this sweep; all but the last side are complete)
        const unsigned rec = h->tl_rec[n];
        h->tl_rec[n] = 0;
        cudaEvent_t* t = h->tl[n];
        float v = 0;
        // [4]: fork -> the solver kernel's end when the one-CTA direct solver ran (t[7] re-recorded
        // after it; the small kernels behind it wait for SM slots beside the side work), else -> t[1]
        if ((rec & 1u) && cudaEventElapsedTime(&v, t[0], t[7]) == cudaSuccess) {
          float w = 0;
          if (v < 1e-3f && cudaEventElapsedTime(&w, t[0], t[1]) == cudaSuccess) v = w;
          h->ov_ms[4] += v;
          ++h->ov_cnt[4];
        }
        if (rec & 12u) {
          float a = 0, b = 0;
          if (cudaEventElapsedTime(&a, t[4], t[5]) == cudaSuccess && cudaEventElapsedTime(&b, t[5], t[6]) == cudaSuccess) {
            h->ov_ms[2] += a;
            h->ov_cnt[2] += (rec & 8u) ? N - 1 : 1;
            h->ov_ms[3] += b;
            ++h->ov_cnt[3];
          }
        }
        if ((rec & 2u) && cudaEventQuery(t[3]) == cudaSuccess) {  // the last mode's side work may still run
          float a = 0, b = 0;
          if (cudaEventElapsedTime(&a, t[0], t[2]) == cudaSuccess && cudaEventElapsedTime(&b, t[2], t[3]) == cudaSuccess) {
            h->ov_ms[0] += a;
            h->ov_cnt[0] += N - 2;
            h->ov_ms[1] += b;
            ++h->ov_cnt[1];
          }
        }
        (void)cudaGetLastError();
      }
      if (mp_timeline()) {
        TK_CUDA(cudaDeviceSynchronize());
        for (int n = 0; n < N; ++n) {
          if (!h->tl[n][0]) continue;
          float a = 0, b = 0, c = 0;
          cudaEventElapsedTime(&a, h->tl[n][0], h->tl[n][1]);
          cudaEventElapsedTime(&b, h->tl[n][0], h->tl[n][2]);
          cudaEventElapsedTime(&c, h->tl[n][0], h->tl[n][3]);
          float d1 = 0, d2 = 0;
          cudaEventElapsedTime(&d1, h->tl[n][4], h->tl[n][5]);
          cudaEventElapsedTime(&d2, h->tl[n][5], h->tl[n][6]);
          std::fprintf(stderr, "mp timeline sweep %d mode %d: eig end %.3f ms, side SpMM end %.3f, side Gram end %.3f; "
                       "late SpMM %.3f, late Gram %.3f\n", s, n, a, b, c, d1, d2);
        }
        (void)cudaGetLastError();  // unrecorded events of the last mode
      }
      eig_check(h, 0, N);
      float ms[4] = {0, 0, 0, ev.ms(4 * N, 4 * N + 1)};
      for (int n = 0; n < N; ++n) {
        ms[0] += ev.ms(4 * n, 4 * n + 1);
        ms[1] += ev.ms(4 * n + 1, 4 * n + 2);
        ms[2] += ev.ms(4 * n + 2, 4 * n + 3);
      }
      if (stage_ms)
        for (int q = 0; q < 4; ++q) stage_ms[4 * s + q] = ms[q];
    }
    return h->eig_unconverged ? TUCKER_E_CONVERGE : TUCKER_OK;
  });
}

int hooi_run(tucker_handle* h, int max_sweeps, double tol, double* fits, int* sweeps_done) {
  return run_until(h, max_sweeps, tol, fits, sweeps_done,
                   [](tucker_handle* hh, double* f) { return hooi_sweep(hh, 1, f, nullptr); });
}

int mp_run(tucker_handle* h, int max_sweeps, double tol, double* fits, int* sweeps_done) {
  return run_until(h, max_sweeps, tol, fits, sweeps_done,
                   [](tucker_handle* hh, double* f) { return mp_sweep(hh, 1, f, nullptr); });
}

// Slice Projection (Figs. 5-6): mode n from the single MP term
// m = n - 1 (cyclic); after every sweep the core and fit (fits[s]) and the core
// norm (gnorms[s], for Delta_G, Eq. 11) -- both nullable.
int sp_sweep(tucker_handle* h, int sweeps, double* fits, double* gnorms, float* stage_ms) {
  if (!h || sweeps < 1 || h->generic) return TUCKER_E_ARG;  // SP: orders 3, 4 (Figs. 5-6)
  return guarded(h, [&]() -> int {
    h->eig_unconverged = false;
    const int N = h->order;
    SweepEvents ev(4 * N + 2);
    for (int s = 0; s < sweeps; ++s) {
      for (int n = 0; n < N; ++n) {
        TK_CUDA(cudaEventRecord(ev.e[4 * n], h->st));
        mp_update(h, n, (n + N - 1) % N, h->slots[2][n], ev.e[4 * n + 1], ev.e[4 * n + 2]);
        TK_CUDA(cudaEventRecord(ev.e[4 * n + 3], h->st));
      }
      TK_CUDA(cudaEventRecord(ev.e[4 * N], h->st));
      const double fit = compute_core(h);  // synchronises (the fit is read on the host)
      TK_CUDA(cudaEventRecord(ev.e[4 * N + 1], h->st));
      TK_CUDA(cudaEventSynchronize(ev.e[4 * N + 1]));
      eig_check(h, 0, N);
      float ms[4] = {0, 0, 0, ev.ms(4 * N, 4 * N + 1)};
      for (int n = 0; n < N; ++n) {
        ms[0] += ev.ms(4 * n, 4 * n + 1);
        ms[1] += ev.ms(4 * n + 1, 4 * n + 2);
        ms[2] += ev.ms(4 * n + 2, 4 * n + 3);
      }
      if (fits) fits[s] = fit;
      if (gnorms) gnorms[s] = std::sqrt(h->last_g2);
      if (stage_ms)
        for (int q = 0; q < 4; ++q) stage_ms[4 * s + q] = ms[q];
    }
    return h->eig_unconverged ? TUCKER_E_CONVERGE : TUCKER_OK;
  });
}

// SP's stop rule (Eq. 11): Delta_G(t) = 1 - ||G^(t-1)|| / ||G^(t)|| < tol
// (||G^(0)|| = 0) or max_sweeps; fits[t] per sweep.
int sp_run(tucker_handle* h, int max_sweeps, double tol, double* fits, int* sweeps_done) {
  if (!h || max_sweeps < 1 || !(tol >= 0)) return TUCKER_E_ARG;
  double gprev = 0.0;
  int t = 0, rc_all = TUCKER_OK;
  while (t < max_sweeps) {
    double fit = 0.0, g = 0.0;
    const int rc = sp_sweep(h, 1, &fit, &g, nullptr);
    if (rc == TUCKER_E_CONVERGE) rc_all = rc;
    else if (rc != TUCKER_OK) return rc;
    if (fits) fits[t] = fit;
    ++t;
    if (g > 0 && 1.0 - gprev / g < tol) break;
    gprev = g;
  }
  if (sweeps_done) *sweeps_done = t;
  return rc_all;
}

int tucker_set_factor(tucker_handle* h, int n, const float* U, int check) {
  if (!h || !U || n < 0 || n >= h->order) return TUCKER_E_ARG;
  const bool on_dev = (h->opts.flags & TUCKER_INPUT_ON_DEVICE) != 0;
  if (!on_dev) {
    if (check) {
      const int rc = validate_factor(U, h->dims[n], h->J[n]);
      if (rc) return rc;
    } else {
      for (int64_t i = 0; i < h->dims[n] * h->J[n]; ++i)
        if (!std::isfinite(U[i])) return TUCKER_E_FACTOR;
    }
  }
  return guarded(h, [&]() -> int {
    TK_CUDA(cudaMemcpyAsync(h->U[n].p, U, h->dims[n] * h->J[n] * sizeof(float),
                            on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->st));
    TK_CUDA(cudaStreamSynchronize(h->st));
    h->G_valid = false;
    memo_invalidate(h, n);
    for (auto& row : h->slots) row[n].valid = false;  // the next solve of mode n starts from U
    return TUCKER_OK;
  });
}

int core_and_fit(tucker_handle* h, float* core_out, float* const* U_out, double* fit_out) {
  if (!h) return TUCKER_E_ARG;
  return guarded(h, [&]() -> int {
    double fit;
    if (h->G_valid && h->Y_mode == h->order - 1) {
      fit = core_from_y(h);  // recompute from the cached Y_(N): cheap, same kernels
    } else {
      fit = compute_core(h);
    }
    const bool od = (h->opts.flags & TUCKER_OUTPUT_ON_DEVICE) != 0;
    const cudaMemcpyKind kind = od ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (core_out) {
      int64_t P = 1;
      for (int n = 0; n < h->order; ++n) P *= h->J[n];
      h->G32.ensure((size_t)P);
      TK_LAUNCH(k_d2f, gridn(P), 256, 0, h->st, h->G64.p, P, h->G32.p);
      TK_CUDA(cudaMemcpyAsync(core_out, h->G32.p, P * sizeof(float), kind, h->st));
    }
    if (U_out)
      for (int n = 0; n < h->order; ++n)
        if (U_out[n])
          TK_CUDA(cudaMemcpyAsync(U_out[n], h->U[n].p, h->dims[n] * h->J[n] * sizeof(float), kind,
                                  h->st));
    TK_CUDA(cudaStreamSynchronize(h->st));
    if (fit_out) *fit_out = fit;
    return TUCKER_OK;
  });
}

int tucker_free(tucker_handle* h) {
  if (!h) return TUCKER_OK;
  cudaSetDevice(h->opts.device);
  if (h->st) cudaStreamSynchronize(h->st);
  const bool own = h->own_stream;
  cudaStream_t st = h->st;
  cudaStream_t st2 = h->st2, sth = h->st_hi;  // MP overlap streams: destroyed after the buffers they allocated
  cudaEvent_t e1 = h->ev_fork, e2 = h->ev_join, e3 = h->ev_eig;
  if (st2) cudaStreamSynchronize(st2);
  if (sth) cudaStreamSynchronize(sth);
  if (h->comm) dist_comm_destroy(h->comm);
  delete h;
  if (st2) {
    cudaStreamSynchronize(st2);
    cudaStreamSynchronize(sth);
    cudaStreamDestroy(st2);
    cudaStreamDestroy(sth);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    cudaEventDestroy(e3);
  }
  if (own && st) cudaStreamDestroy(st);
  return TUCKER_OK;
}

int tucker_debug_ttmc(tucker_handle* h, int mode, float* Y_out) {
  if (!h || !Y_out || mode < 0 || mode >= h->order) return TUCKER_E_ARG;
  return guarded(h, [&]() -> int {
    project_hooi(h, mode, false);
    h->G_valid = false;
    const int64_t rows = h->Y.rows, cols = h->Y.cols;
    h->Ytmp.ensure((size_t)(rows * cols));
    TK_LAUNCH(k_combine, gridn(rows * cols), 256, 0, h->st, h->Y.hi, h->Y.lo, rows, cols, h->Y.ld,
              h->Ytmp.p);
    const bool od = (h->opts.flags & TUCKER_OUTPUT_ON_DEVICE) != 0;
    TK_CUDA(cudaMemcpyAsync(Y_out, h->Ytmp.p, rows * cols * sizeof(float),
                            od ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->st));
    TK_CUDA(cudaStreamSynchronize(h->st));
    return TUCKER_OK;
  });
}

int tucker_debug_gram(tucker_handle* h, int algo, int mode, double* S_out) {
  if (!h || !S_out || mode < 0 || mode >= h->order || algo < 0 || algo > 1) return TUCKER_E_ARG;
  if (algo == 1 && h->generic) return TUCKER_E_ARG;
  return guarded(h, [&]() -> int {
    Split A;
    const bool sparse = algo == 1 && mp_use_sparse(h, mode, -1);
    if (algo == 0) {
      project_hooi(h, mode, false);
      h->G_valid = false;
      A = h->Y;
    } else if (!sparse) {
      A = build_mp_w(h, mode);
    }
    const int64_t d = h->dims[mode];
    const int64_t lds = ensure_S(h, d);
    if (sparse) build_mp_gram_sparse(h, mode, -1);
    else gram_syrk(A, h->S.p, lds, h->gram, h->st);
    const bool od = (h->opts.flags & TUCKER_OUTPUT_ON_DEVICE) != 0;
    TK_CUDA(cudaMemcpy2DAsync(S_out, d * sizeof(double), h->S.p, lds * sizeof(double), d * sizeof(double), d,
                              od ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->st));
    TK_CUDA(cudaStreamSynchronize(h->st));
    return TUCKER_OK;
  });
}

int tucker_debug_gram_rows(tucker_handle* h, int algo, int mode, int nrows, const int64_t* rows, double* out) {
  if (!h || !rows || !out || nrows < 1 || mode < 0 || mode >= h->order || algo < 0 || algo > 1) return TUCKER_E_ARG;
  if (algo == 1 && h->generic) return TUCKER_E_ARG;
  for (int r = 0; r < nrows; ++r)
    if (rows[r] < 0 || rows[r] >= h->dims[mode]) return TUCKER_E_ARG;
  return guarded(h, [&]() -> int {
    const int64_t d = h->dims[mode];
    const int64_t lds = ensure_S(h, d);
    if (algo == 0) {
      project_hooi(h, mode, false);
      h->G_valid = false;
      gram_syrk(h->Y, h->S.p, lds, h->gram, h->st);
    } else if (mp_use_sparse(h, mode, -1)) {
      build_mp_gram_sparse(h, mode, -1);
    } else {
      gram_syrk(build_mp_w(h, mode), h->S.p, lds, h->gram, h->st);
    }
    for (int r = 0; r < nrows; ++r)
      TK_CUDA(cudaMemcpyAsync(out + (int64_t)r * d, h->S.p + rows[r] * lds, d * sizeof(double),
                              cudaMemcpyDeviceToHost, h->st));
    TK_CUDA(cudaStreamSynchronize(h->st));
    return TUCKER_OK;
  });
}

int tucker_debug_eig(tucker_handle* h, int d, int J, const double* S, float* U_out,
                     double* evals_out) {
  if (!h || !S || !U_out || d < 1 || J < 1 || J > d || J > kMaxJ) return TUCKER_E_ARG;
  return guarded(h, [&]() -> int {
    const int64_t lds = ensure_S(h, d);
    const bool od = (h->opts.flags & TUCKER_OUTPUT_ON_DEVICE) != 0;
    TK_CUDA(cudaMemcpy2DAsync(h->S.p, lds * sizeof(double), S, (size_t)d * sizeof(double),
                              (size_t)d * sizeof(double), d,
                              od ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->st));
    h->scratch_slot.valid = false;
    h->eig_unconverged = false;
    solve_eig(h, d, J, h->scratch_slot);
    h->Ytmp.ensure((size_t)d * J);
    canon_to_f32(h->V.p, J, d, J, h->Ytmp.p, h->st);
    TK_CUDA(cudaMemcpyAsync(U_out, h->Ytmp.p, (size_t)d * J * sizeof(float),
                            od ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->st));
    TK_CUDA(cudaStreamSynchronize(h->st));
    eig_check(h);
    if (evals_out)
      TK_CUDA(cudaMemcpy(evals_out, h->theta_d.p, J * sizeof(double), cudaMemcpyDeviceToHost));
    return h->eig_unconverged ? TUCKER_E_CONVERGE : TUCKER_OK;
  });
}

int tucker_debug_smalldense(int mode, int k, const double* in, double* out, double* theta,
                            int* sweeps, int max_sweeps, double shift) {
  if (!in || !out || k < 1 || k > kMaxBlock || mode < 0 || mode > 2) return TUCKER_E_ARG;
  return guarded(nullptr, [&]() -> int {
    DBuf<double> din((size_t)k * k), dout((size_t)k * k), dth((size_t)k);
    DBuf<int> di(8);
    TK_CUDA(cudaMemcpy(din.p, in, (size_t)k * k * sizeof(double), cudaMemcpyHostToDevice));
    eig_unit(mode, din.p, k, dout.p, dth.p, di.p, max_sweeps, shift, 0);
    TK_CUDA(cudaDeviceSynchronize());
    TK_CUDA(cudaMemcpy(out, dout.p, (size_t)k * k * sizeof(double), cudaMemcpyDeviceToHost));
    if (theta) TK_CUDA(cudaMemcpy(theta, dth.p, (size_t)k * sizeof(double), cudaMemcpyDeviceToHost));
    if (sweeps) TK_CUDA(cudaMemcpy(sweeps, di.p, (mode >= 1 ? 8 : 1) * sizeof(int), cudaMemcpyDeviceToHost));
    return TUCKER_OK;
  });
}

int tucker_debug_product(int d, int n, const double* S, const double* Y, double alpha, double gamma,
                         const double* D, double* out) {
  if (!S || !Y || !out || d < 1 || n < 1 || n > kMaxBlock) return TUCKER_E_ARG;
  return guarded(nullptr, [&]() -> int {
    DBuf<double> dS((size_t)d * d), dY((size_t)d * n), dD((size_t)d * n), dO((size_t)d * n);
    TK_CUDA(cudaMemcpy(dS.p, S, (size_t)d * d * sizeof(double), cudaMemcpyHostToDevice));
    TK_CUDA(cudaMemcpy(dY.p, Y, (size_t)d * n * sizeof(double), cudaMemcpyHostToDevice));
    if (D) TK_CUDA(cudaMemcpy(dD.p, D, (size_t)d * n * sizeof(double), cudaMemcpyHostToDevice));
    TK_CUDA(cudaMemset(dO.p, 0xff, (size_t)d * n * sizeof(double)));
    if (alpha == 12345.0) {  // debug: determinism of two back-to-back products
      out[0] = eig_unit_mv_repeat(dS.p, dY.p, d, n);
      return TUCKER_OK;
    }
    eig_unit_mv(dS.p, dY.p, d, n, alpha, dO.p, D ? gamma : 0.0, dD.p, 0);
    TK_CUDA(cudaDeviceSynchronize());
    TK_CUDA(cudaMemcpy(out, dO.p, (size_t)d * n * sizeof(double), cudaMemcpyDeviceToHost));
    return TUCKER_OK;
  });
}

int tucker_debug_product_time(int d, int n, int reps, double* us) {
  if (!us || d < 1 || n < 1 || n > kMaxBlock || reps < 1) return TUCKER_E_ARG;
  return guarded(nullptr, [&]() -> int {
    *us = eig_unit_mv_time(d, n, reps);
    return TUCKER_OK;
  });
}

int tucker_time_ttmc(tucker_handle* h, int mode, int reps, float* ms_out) {
  if (!h || !ms_out || mode < 0 || mode >= h->order || reps < 1) return TUCKER_E_ARG;
  return guarded(h, [&]() -> int {
    const bool tr = prod_J_except(h, mode) < h->dims[mode] && h->J[mode] <= kMaxBlock;
    // the sweep's path: a sibling mode of the partial-contraction reuse reads the Z its root mode kept
    for (auto& m : h->memo)
      if (m.csf >= 0 && m.sib == mode && !m.valid) project_hooi(h, m.root, false);
    project_hooi(h, mode, tr);  // untimed: buffers, first-touch
    SweepEvents ev(2);
    TK_CUDA(cudaEventRecord(ev.e[0], h->st));
    for (int r = 0; r < reps; ++r) project_hooi(h, mode, tr);
    TK_CUDA(cudaEventRecord(ev.e[1], h->st));
    TK_CUDA(cudaEventSynchronize(ev.e[1]));
    *ms_out = ev.ms(0, 1) / (float)reps;
    h->G_valid = false;
    return TUCKER_OK;
  });
}

int tucker_csf_layout(tucker_handle* h, int64_t* out) {
  if (!h || !out || h->generic) return TUCKER_E_ARG;
  for (int n = 0; n < h->order; ++n) {
    const Csf& c = *h->csfs[h->hooi_csf[n]];
    int64_t* o = out + 8 * n;
    o[0] = c.root;
    o[1] = c.mid0;
    o[2] = c.order == 4 ? c.mid1 : -1;
    o[3] = c.leaf;
    o[4] = c.nfib;
    o[5] = c.order == 4 ? c.nnode : 0;
    o[6] = c.nnz;
    o[7] = c.I_root;
  }
  return TUCKER_OK;
}

int tucker_csf_stats(tucker_handle* h, int64_t* out) {
  if (!h || !out || h->generic) return TUCKER_E_ARG;
  for (int n = 0; n < h->order; ++n) {
    const Csf& c = *h->csfs[h->hooi_csf[n]];
    out[4 * n] = c.nfib;
    out[4 * n + 1] = c.nnz;
    out[4 * n + 2] = c.nvfib;   // 0: no work plan (one CTA per slice)
    out[4 * n + 3] = c.nunits;
  }
  return TUCKER_OK;
}

int tucker_hosvd(tucker_handle* h, unsigned mode_mask) {
  if (!h || (mode_mask >> h->order) != 0 || h->generic) return TUCKER_E_ARG;
  return guarded(h, [&]() -> int {
    h->eig_unconverged = false;
    for (int n = 0; n < h->order; ++n) {
      if (!((mode_mask >> n) & 1u)) continue;
      // an ordering with leaf n: each fiber is one column of X_(n)
      const int r = (n + 1) % h->order;
      const Csf& c = *h->csfs[h->mp_csf[r][n]];
      const int64_t d = h->dims[n];
      const int J = (int)h->J[n];
      const int64_t lds = ensure_S(h, d);
      TK_CUDA(cudaMemsetAsync(h->S.p, 0, (size_t)(d * lds) * sizeof(double), h->st));
      int64_t f0 = 0, f1 = c.nfib;
      if (h->sharded) {  // equal fiber ranges (work ~ pairs per fiber, uniform enough for a one-off)
        f0 = c.nfib * h->opts.rank / h->opts.world;
        f1 = c.nfib * (h->opts.rank + 1) / h->opts.world;
      }
      sparse_gram(c, f0, f1, h->S.p, lds, h->st);
      if (h->sharded) dist_allreduce_f64(h->comm, h->S.p, d * lds, h->st);
      h->scratch_slot.valid = false;
      memo_invalidate(h, n);
      solve_eig(h, d, J, h->scratch_slot, h->U[n].p);
      canon_to_f32(h->V.p, J, d, J, h->U[n].p, h->st);
      TK_CUDA(cudaStreamSynchronize(h->st));
      eig_check(h);
    }
    h->G_valid = false;
    return h->eig_unconverged ? TUCKER_E_CONVERGE : TUCKER_OK;
  });
}

int tucker_nccl_unique_id(void* id_out) {
  if (!id_out) return TUCKER_E_ARG;
  return guarded(nullptr, [&]() -> int {
    dist_unique_id(id_out);
    return TUCKER_OK;
  });
}

int tucker_shard_bounds(const double* work, int64_t n, int world, int64_t* bounds) {
  if (!bounds || world < 1 || n < 0 || (n > 0 && !work)) return TUCKER_E_ARG;
  for (int64_t i = 0; i < n; ++i)
    if (!(work[i] >= 0)) return TUCKER_E_ARG;
  shard_bounds(work, n, world, bounds);
  return TUCKER_OK;
}

int tucker_set_allreduce(tucker_handle* h, void* fn, void* user) {
  if (!h || !fn || !h->comm || !(h->opts.flags & TUCKER_HOST_COLLECTIVES)) return TUCKER_E_ARG;
  dist_comm_set_callback(h->comm, fn, user);
  return TUCKER_OK;
}

int tucker_shard_info(tucker_handle* h, int64_t* out) {
  if (!h || !out || h->generic) return TUCKER_E_ARG;
  const int N = h->order;
  for (int n = 0; n < N; ++n) {
    const Csf& c = *h->csfs[h->hooi_csf[n]];
    out[2 * n] = h->sharded ? h->hooi_lo[n] : 0;
    out[2 * n + 1] = h->sharded ? h->hooi_hi[n] : c.I_root;
    for (int m = 0; m < N; ++m) {
      int64_t* o = out + 2 * N + 2 * (n * N + m);
      if (m == n) {
        o[0] = o[1] = 0;
        continue;
      }
      const Csf& t = *h->csfs[h->mp_csf[n][m]];
      o[0] = h->sharded ? h->mp_lo[n][m] : 0;
      o[1] = h->sharded ? h->mp_hi[n][m] : t.I_mid0 * t.I_mid1;
    }
  }
  return TUCKER_OK;
}

int tucker_mp_overlap_times(tucker_handle* h, double* ms, int64_t* counts, int reset) {
  if (!h || !ms || !counts) return TUCKER_E_ARG;
  for (int q = 0; q < 5; ++q) {
    ms[q] = h->ov_ms[q];
    counts[q] = h->ov_cnt[q];
    if (reset) {
      h->ov_ms[q] = 0;
      h->ov_cnt[q] = 0;
    }
  }
  return TUCKER_OK;
}

int tucker_stats(tucker_handle* h, int64_t* stats, int reset) {
  if (!h || !stats) return TUCKER_E_ARG;
  stats[0] = h->launches;
  stats[1] = h->eig.stat_outer - h->stat_outer0;
  stats[2] = h->eig.stat_matvec - h->stat_matvec0;
  stats[3] = h->eig.stat_sweeps - h->stat_sweeps0;
  stats[4] = gram_path_id();
  {
    long long pf[13] = {0};
    if (h->eig.fprof.p && h->eig.fprof_init) {
      if (cudaMemcpy(pf, h->eig.fprof.p, sizeof(pf), cudaMemcpyDeviceToHost) != cudaSuccess)
        return TUCKER_E_CUDA;
    }
    for (int i = 0; i < 13; ++i) stats[5 + i] = pf[i] - h->prof0[i];
    if (reset)
      for (int i = 0; i < 13; ++i) h->prof0[i] = pf[i];
  }
  if (reset) {
    h->launches = 0;
    h->stat_outer0 = h->eig.stat_outer;
    h->stat_matvec0 = h->eig.stat_matvec;
    h->stat_sweeps0 = h->eig.stat_sweeps;
  }
  return TUCKER_OK;
}

}  // extern "C"
