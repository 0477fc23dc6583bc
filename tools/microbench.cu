// Development microbenchmarks (not part of the library): grid.sync latency,
// DMMA (fp64 tensor) and DFMA throughput on one B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench.cu && /tmp/mb
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_gsync(int n, int* sink) {
  for (int i = 0; i < n; ++i) cg::this_grid().sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) *sink = n;
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
__global__ void k_dfma(int n, double* out) {
  double x[8];
  for (int t = 0; t < 8; ++t) x[t] = threadIdx.x + t;
  const double a = 1.0000001, b = 1e-9;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int t = 0; t < 8; ++t) x[t] = fma(x[t], a, b);
  double s = 0;
  for (int t = 0; t < 8; ++t) s += x[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_smem_rt(int n, double* out) {  // dependent smem + barrier latency
  __shared__ double buf[1024];
  buf[threadIdx.x] = threadIdx.x;
  __syncthreads();
  double v = 0;
  for (int i = 0; i < n; ++i) {
    v += buf[(threadIdx.x + i) & 511];
    __syncthreads();
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = v;
}

int main_tp();
int main_lat();
int main() { main_lat(); return main_tp(); }
int main_tp() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int* sink;
  double* out;
  cudaMalloc(&sink, 4);
  cudaMalloc(&out, 148 * 1024 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int threads : {256, 512}) {
    int n = 2000;
    void* args[] = {&n, &sink};
    cudaLaunchCooperativeKernel((void*)k_gsync, nsm, threads, args, 0, 0);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k_gsync, nsm, threads, args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("grid.sync %d CTAs x %d thr: %.3f us/sync (%s)\n", nsm, threads, ms * 1e3 / n,
           cudaGetErrorString(cudaGetLastError()));
  }
  {
    int n = 4096;
    for (int warps : {4, 8, 16}) {
      k_dmma<<<nsm, 32 * warps>>>(n, out);
      cudaEventRecord(e0);
      k_dmma<<<nsm, 32 * warps>>>(n, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 256 * 8 * (double)n * warps * nsm;
      printf("DMMA %2d warps/SM: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
    }
  }
  {
    int n = 4096;
    for (int thr : {256, 512, 1024}) {
      k_dfma<<<nsm, thr>>>(n, out);
      cudaEventRecord(e0);
      k_dfma<<<nsm, thr>>>(n, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 8 * (double)n * thr * nsm;
      printf("DFMA %4d thr/SM: %.2f TFLOP/s\n", thr, fl / ms / 1e9);
    }
  }
  {
    int n = 20000;
    k_smem_rt<<<1, 512>>>(n, out);
    cudaEventRecord(e0);
    k_smem_rt<<<1, 512>>>(n, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("smem load + __syncthreads (512 thr): %.1f ns/iter\n", ms * 1e6 / n);
  }
  return 0;
}

// dependent-chain latencies (single warp), cycles per op
__global__ void k_lat(double* out, float* outf, long long* cyc, int n) {
  double a = out[0], b = 1.0000001;
  float fa = outf[0], fb = 1.0001f;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, 1e-9);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) fa = fmaf(fa, fb, 1e-9f);
  long long t2 = clock64();
  double r = a;
  for (int i = 0; i < n; ++i) r = 1.0 / (r + 1.0);
  long long t3 = clock64();
  double q = a;
  for (int i = 0; i < n; ++i) q = sqrt(q + 1.0);
  long long t4 = clock64();
  __shared__ double sm[64];
  sm[threadIdx.x] = a;
  __syncwarp();
  int idx = threadIdx.x;
  double acc = 0;
  for (int i = 0; i < n; ++i) { acc += sm[idx]; idx = (int)acc & 31; }
  long long t5 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / n; cyc[1] = (t2 - t1) / n; cyc[2] = (t3 - t2) / n; cyc[3] = (t4 - t3) / n;
    cyc[4] = (t5 - t4) / n;
  }
  out[threadIdx.x] = a + r + q + acc;
  outf[threadIdx.x] = fa;
}
int main_lat() {
  double* o; float* of; long long* c;
  cudaMalloc(&o, 64 * 8); cudaMalloc(&of, 64 * 4); cudaMalloc(&c, 64);
  cudaMemset(o, 0, 64 * 8); cudaMemset(of, 0, 64 * 4);
  k_lat<<<1, 32>>>(o, of, c, 1000);
  long long h[5];
  cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
  printf("latency cycles: DFMA %lld  FFMA %lld  DDIV(+add) %lld  DSQRT(+add) %lld  LDS-dep %lld\n", h[0], h[1], h[2], h[3], h[4]);
  return 0;
}
