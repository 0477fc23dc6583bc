// Standalone check of tcgen05.mma kind::tf32 with MN-major, 128B-swizzled
// smem operands: D(128 x N) = A(128 x K) B(N x K)^T for K = 8 (one MMA) and 32 (four).
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_0711_2023_b200/csrc/tc_ptx.cuh"
using namespace tk;
constexpr int M = 128, N = 64, K = 32, KGR = K / 8;
__device__ __forceinline__ uint32_t mn_sw128(int mn, int k) {
  const int atom = mn >> 5, inner = mn & 31, kg = k >> 3, kr = k & 7;
  return (uint32_t)(atom * (KGR * 1024) + kg * 1024 + kr * 128 + ((((inner >> 2) ^ kr) << 4) | ((inner & 3) << 2)));
}
__device__ __forceinline__ uint32_t k_sw128(int mn, int k) {  // K-major, K = 32 per 128 B row
  return (uint32_t)((mn >> 3) * 1024 + (mn & 7) * 128 + ((((k >> 2) ^ (mn & 7)) << 4) | ((k & 3) << 2)));
}
__global__ void k_test(const float* A, const float* B, float* D, int variant) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* sa = sm;
  uint8_t* sb = sm + 4 * KGR * 1024;
  for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
    const int m = e / K, k = e % K;
    *reinterpret_cast<float*>(sa + (variant == 8 ? k_sw128(m, k) : mn_sw128(m, k))) = A[m * K + k];
  }
  for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
    const int n = e / K, k = e % K;
    *reinterpret_cast<float*>(sb + (variant == 8 ? k_sw128(n, k) : mn_sw128(n, k))) = B[n * K + k];
  }
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&slot)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t amaj = (variant & 1) ? 1u : 0u, bmaj = (variant & 2) ? 1u : 0u;  // variant 8: K-major
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (amaj << 15) | (bmaj << 16) |
                         ((uint32_t)N >> 3 << 17) | ((uint32_t)M >> 4 << 24);
  const bool swap = variant & 4;
  if (threadIdx.x == 0) {
    const uint32_t a0 = tc::smem_u32(sa), b0 = tc::smem_u32(sb);
    const uint32_t atom = KGR * 1024;
    if (variant == 8) {
      for (int g = 0; g < KGR; ++g)
        tc::umma_tf32(tmem, tc::sw128_desc(a0 + g * 32), tc::sw128_desc(b0 + g * 32), idesc, g > 0 ? 1u : 0u);
    } else
    for (int g = 0; g < KGR; ++g) {
      const uint32_t lbo = swap ? 1024 : atom, sbo = swap ? atom : 1024;
      tc::umma_tf32(tmem, tc::sw128_desc_lbo_sbo(a0 + g * 1024, lbo, sbo),
                    tc::sw128_desc_lbo_sbo(b0 + g * 1024, lbo, sbo), idesc, g > 0 ? 1u : 0u);
    }
    tc::umma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  if (threadIdx.x < 128) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    for (int nb = 0; nb < N / 32; ++nb) {
      float v[32];
      tc::tmem_ld32(tmem + ((uint32_t)(32 * w) << 16) + 32 * nb, v);
      tc::tmem_wait_ld();
      for (int j = 0; j < 32; ++j) D[(32 * w + l) * N + 32 * nb + j] = v[j];
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}
int main(int argc, char** argv) {
  std::vector<float> A(M * K), B(N * K), D(M * N), R(M * N);
  for (int i = 0; i < M * K; ++i) A[i] = (float)((i * 7 % 13) - 6) / 8.f;
  for (int i = 0; i < N * K; ++i) B[i] = (float)((i * 5 % 11) - 5) / 4.f;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[n * K + k];
      R[m * N + n] = (float)s;
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 4 * KGR * 1024 + 2 * KGR * 1024 + 1024;
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int variant = atoi(argv[1]); variant <= atoi(argv[1]); ++variant) {
    cudaMemset(dD, 0, D.size() * 4);
    k_test<<<1, 256, smem>>>(dA, dB, dD, variant);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0, ref = 0;
    for (int i = 0; i < M * N; ++i) { err = fmax(err, fabs(D[i] - R[i])); ref = fmax(ref, fabs(R[i])); }
    printf("variant %d (a_mn %d b_mn %d swap_lbo_sbo %d): %s max err %.3g (ref %.3g) D[0..3] %g %g %g %g vs %g %g %g %g\n",
           variant, variant & 1, (variant >> 1) & 1, (variant >> 2) & 1, cudaGetErrorString(e), err, ref,
           D[0], D[1], D[2], D[3], R[0], R[1], R[2], R[3]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
