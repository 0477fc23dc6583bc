// fp64 latency microbenchmark (one warp): dependent DFMA, DADD, double shfl, sqrt, division,
// FFMA for comparison, and a __syncthreads round with 1024 threads.  nvcc -arch=sm_100a
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b, int iters) {
  double x = a, y = b;
  float fx = (float)a;
  long long t0, t1;
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, b, a);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) y = y + x * 0.0 + 1e-300, y = y + 1e-300;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = sqrt(x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = 2.0 / (x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) fx = fmaf(fx, (float)b, (float)a);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = t1 - t0;
  __shared__ double sh[1024];
  sh[threadIdx.x] = x;
  __syncthreads();
  int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = sh[idx]; idx = ((int)x & 0) + ((idx + 1) & 1023); }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[7] = t1 - t0;
  out[threadIdx.x] = x + y + fx;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64 * 8);
  const int it = 1000;
  for (int nt : {32, 1024}) {
    k<<<1, nt>>>(o, c, 0.5, 0.999, it);
    long long h[8];
    cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    printf("threads %d cycles/op: dfma %.1f dadd(2/it) %.1f shfl64 %.1f sqrt %.1f div %.1f ffma %.1f syncthreads %.1f lds64-chain %.1f\n", nt,
           h[0] / (double)it, h[1] / (2.0 * it), h[2] / (double)it, h[3] / (double)it, h[4] / (double)it, h[5] / (double)it,
           h[6] / (double)it, h[7] / (double)it);
  }
  return 0;
}
