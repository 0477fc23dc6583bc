// Measured compute peaks used as roofline denominators (bench.py):
//   FFMA  fp32 CUDA-core FMA throughput (independent chains, all SMs)
//   DMMA  fp64 tensor-core mma.sync.m8n8k4 throughput
//   TF32  tcgen05.mma kind::tf32 issue-bound throughput: one CTA per SM, operands
//         resident in shared memory (no loads), M = 128, N = 256, K = 8 per
//         instruction, fp32 accumulators in TMEM -- the tensor pipe's own ceiling
// Output: one JSON object on stdout.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks tools/peaks.cu -lcuda && /tmp/peaks
#include <cuda.h>
#include <cstdio>
#include <cstdint>

#include "../paper_0711_2023_b200/csrc/tc_ptx.cuh"

__global__ void k_ffma(int n, float* out) {
  float x[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) x[t] = threadIdx.x * 1e-3f + t;
  const float a = 1.0000001f, b = 1e-9f;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int t = 0; t < 16; ++t) x[t] = fmaf(x[t], a, b);
  float s = 0;
#pragma unroll
  for (int t = 0; t < 16; ++t) s += x[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dmma(int n, double* out) {
  double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
  double c[8][2] = {};
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_mma_tf32(int n, float* out) {  // legacy warp-level mma.sync.m16n8k8 tf32
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[8][4] = {};
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[t][0]), "+f"(c[t][1]), "+f"(c[t][2]), "+f"(c[t][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// A: 128 x 32 tf32 (16 KB), B: 256 x 32 tf32 (32 KB), K-major SW128; D: 128 x 256 fp32 in TMEM
constexpr int TN = 256;
__global__ void __launch_bounds__(128) k_tf32(int n, float* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  for (int o = threadIdx.x * 16; o < (128 + TN) * 128; o += 128 * 16)
    *reinterpret_cast<float4*>(sm + o) = make_float4(1e-3f, 2e-3f, 3e-3f, 4e-3f);
  if (threadIdx.x == 0) {
    tk::tc::mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tk::tc::smem_u32(&slot)), "r"(TN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tk::tc::tc_fence_before();
  __syncthreads();
  tk::tc::tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t a = tk::tc::smem_u32(sm), b = a + 128 * 128;
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TN >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
#pragma unroll
      for (int g = 0; g < 4; ++g)
        tk::tc::umma_tf32(tmem, tk::tc::sw128_desc(a + 32 * g), tk::tc::sw128_desc(b + 32 * g), IDESC,
                          (i | g) ? 1u : 0u);
    }
    tk::tc::umma_commit(&bar);
  }
  tk::tc::mbar_wait(&bar, 0);
  tk::tc::tc_fence_after();
  float v[32];
  tk::tc::tmem_ld32(tmem + ((uint32_t)(32 * (threadIdx.x >> 5)) << 16), v);
  tk::tc::tmem_wait_ld();
  out[blockIdx.x * 128 + threadIdx.x] = v[0];
  tk::tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TN));
}

template <typename F>
float time_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* outf;
  double* outd;
  cudaMalloc(&outf, 148 * 1024 * 8);
  cudaMalloc(&outd, 148 * 1024 * 8);
  double ffma = 0, dmma = 0, tf32 = 0;
  for (int thr : {512, 1024}) {
    const int n = 8192;
    const float ms = time_ms([&] { k_ffma<<<2 * nsm, thr>>>(n, outf); });
    const double t = 2.0 * 16 * (double)n * thr * 2 * nsm / ms / 1e9;
    if (t > ffma) ffma = t;
  }
  for (int warps : {8, 16}) {
    const int n = 4096;
    const float ms = time_ms([&] { k_dmma<<<nsm, 32 * warps>>>(n, outd); });
    const double t = 2.0 * 256 * 8 * (double)n * warps * nsm / ms / 1e9;
    if (t > dmma) dmma = t;
  }
  double mma_tf32 = 0;
  for (int warps : {8, 16, 32}) {
    const int n = 4096;
    const float ms = time_ms([&] { k_mma_tf32<<<nsm, 32 * warps>>>(n, outf); });
    const double t = 2.0 * 16 * 8 * 8 * 8 * (double)n * warps * nsm / ms / 1e9;
    if (t > mma_tf32) mma_tf32 = t;
  }
  {
    const int smem = (128 + TN) * 128 + 1024;
    cudaFuncSetAttribute(k_tf32, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int n = 20000;
    const float ms = time_ms([&] { k_tf32<<<nsm, 128, smem>>>(n, outf); });
    tf32 = 2.0 * 128 * TN * 32 * (double)n * nsm / ms / 1e9;
  }
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"ffma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"tcgen05_tf32_tflops\": %.1f, "
         "\"mma_sync_tf32_tflops\": %.1f, \"sms\": %d, \"err\": \"%s\"}\n",
         ffma, dmma, tf32, mma_tf32, nsm, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
