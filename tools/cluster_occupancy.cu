// How many clusters of a given size can be co-resident on this GPU (one CTA per SM, ~200 KB smem):
// the multicast-cluster GEMM of DESIGN.md §11 loses SMs if 148 is not covered by whole clusters.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cluster_occ tools/cluster_occupancy.cu && /tmp/cluster_occ
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dummy(int* p) {
  extern __shared__ int s[];
  if (p) p[threadIdx.x] = s[threadIdx.x];
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
    printf("SMs %d  cluster %2d: max active clusters %3d -> %3d CTAs (%s)\n", sms, cs, n, n * cs,
           e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  }
  return 0;
}
