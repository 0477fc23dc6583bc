// Throughput of the legacy warp-level mma.sync.m16n8k8 tf32 (fp32 accumulate)
// on sm_100a, register operands only (upper bound for an mma.sync Kronecker).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_mma(int n, float* out) {
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
  if (s == 12345.f) out[0] = s;
}
int main() {
  float* out;
  cudaMalloc(&out, 4);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    const int n = 20000;
    k_mma<<<nsm, 32 * warps>>>(100, out);
    cudaEventRecord(e0);
    k_mma<<<nsm, 32 * warps>>>(n, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 16 * 8 * 8 * 8.0 * n * warps * nsm;
    printf("mma.sync m16n8k8 tf32 %2d warps/SM: %.1f TFLOP/s\n", warps, fl / ms / 1e9);
  }
  return 0;
}
