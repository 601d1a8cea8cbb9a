// How many thread-block clusters of size 2/4/8/16 can be co-resident on this GPU for a kernel
// with ~227 KB of dynamic shared memory (one CTA per SM), i.e. how many SMs a cluster-multicast
// GEMM could use.  nvcc -gencode arch=compute_100a,code=sm_100a -o cluster_occupancy cluster_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(int* p) {
  extern __shared__ int s[];
  s[threadIdx.x] = threadIdx.x;
  if (p) p[blockIdx.x] = s[0];
}

int main() {
  const int smem = 227 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(320);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: max active clusters %3d -> %3d of %d SMs busy (%s)\n", cs, n, n * cs, sms,
           cudaGetErrorString(e));
  }
  return 0;
}
