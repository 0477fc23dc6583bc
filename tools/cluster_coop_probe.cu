// Can k_eig_fused-like kernels (512 threads, ~200 KB smem, 1 CTA/SM) run as a
// cooperative launch in thread-block clusters?  Reports the co-resident
// cluster count per cluster size and runs a cooperative cluster launch with a
// grid.sync() + a cluster barrier.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void k_probe(int* out) {
  extern __shared__ double sm[];
  cg::grid_group grid = cg::this_grid();
  cg::cluster_group cl = cg::this_cluster();
  sm[threadIdx.x] = threadIdx.x;
  cl.sync();
  grid.sync();
  if (threadIdx.x == 0) atomicAdd(out, 1);
}
int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int* d;
  cudaMalloc(&d, 4);
  for (int cs : {1, 2, 4, 8}) {
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cfg.gridDim = dim3(cs);
    int ncl = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, k_probe, &cfg);
    const int grid = ncl * cs;
    cfg.gridDim = dim3(grid);
    cudaMemset(d, 0, 4);
    cudaError_t e2 = cudaLaunchKernelEx(&cfg, k_probe, d);
    cudaError_t e3 = cudaDeviceSynchronize();
    int h = 0;
    cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("cluster %d: max active clusters %d (%s) -> grid %d of %d SMs; coop launch %s / %s, CTAs done %d\n", cs, ncl,
           cudaGetErrorString(e), grid, nsm, cudaGetErrorString(e2), cudaGetErrorString(e3), h);
    if (e3 != cudaSuccess) return 1;
  }
  return 0;
}
