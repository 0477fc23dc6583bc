// microbenchmark: shared-memory wavefronts of warp-uniform vs lane-distinct LDS.128 / LDS.32
// (decides the register tile of the order-4 SpTTMc GEMM form).  nvcc -arch=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int iters) {
  __shared__ __align__(16) float s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 1e-3f;
  __syncthreads();
  float a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    const int base = (it * 36) & 2047;
    float4 v;
    if (MODE == 0) v = *reinterpret_cast<const float4*>(s + (base & ~3));                 // uniform 128-bit
    else if (MODE == 1) v = *reinterpret_cast<const float4*>(s + ((base & ~3) + 4 * lane)); // distinct 128-bit
    else if (MODE == 2) { v.x = s[base]; v.y = s[base + 1]; v.z = s[base + 2]; v.w = s[base + 3]; }  // uniform 32-bit x4
    else { const int o = (base + lane * 5) & 4095; v.x = s[o]; v.y = s[o + 1]; v.z = s[o + 2]; v.w = s[o + 3]; }
    a0 = fmaf(v.x, a0, v.y); a1 = fmaf(v.y, a1, v.z); a2 = fmaf(v.z, a2, v.w); a3 = fmaf(v.w, a3, v.x);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 1 << 16;
  void (*fns[4])(float*, int) = {k<0>, k<1>, k<2>, k<3>};
  const char* nm[4] = {"uniform LDS.128", "distinct LDS.128", "uniform LDS.32x4", "distinct LDS.32x4"};
  for (int m = 0; m < 4; ++m) {
    fns[m]<<<148 * 4, 256>>>(o, 64);
    cudaEventRecord(e0);
    fns[m]<<<148 * 4, 256>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double warp_loads = 148.0 * 4 * 8 * iters;  // warp-level load instructions (x1 or x4)
    printf("%-20s %.3f ms  %.3f ns per warp-load per SM\n", nm[m], ms, ms * 1e6 / (warp_loads / 148));
  }
  return 0;
}
