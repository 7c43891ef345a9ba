// How many thread-block clusters of a given size can be co-resident with one
// ~200 KB-smem CTA per SM (cudaOccupancyMaxActiveClusters), and a measured
// DSMEM cluster-barrier round trip.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void kprobe(long long* out) {
  extern __shared__ int smem[];
  cg::cluster_group cl = cg::this_cluster();
  smem[threadIdx.x] = threadIdx.x;
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < 16; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / 16;
}

int main() {
  const size_t smem = 200 * 1024;
  cudaFuncSetAttribute(kprobe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kprobe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  long long* out;
  cudaMalloc(&out, 4096 * 8);
  for (int cs : {2, 4, 6, 8, 9, 12, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 8);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kprobe, &cfg);
    long long h = -1;
    if (e == cudaSuccess && n >= 8) {
      cudaLaunchKernelEx(&cfg, kprobe, out);
      cudaDeviceSynchronize();
      cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    }
    printf("cluster %2d: max active clusters %3d (%s) -> CTAs %4d; cluster.sync %lld cycles\n", cs, n,
           cudaGetErrorString(e), n * cs, h);
  }
  return 0;
}
