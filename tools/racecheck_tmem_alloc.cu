// Minimal reproducer for the racecheck report on the CTA-pair GEMM (profiles/r01h_sanitizer.txt):
// a cluster of 2 CTAs where one warp of each CTA performs tcgen05.alloc.cta_group::2 into a shared-memory
// slot, the pair synchronises (barrier.cluster release/acquire) and every thread reads the slot -- the
// exact setup sequence of fp8_gemm_kernel, with no GEMM.  Variant 1 is the same with cta_group::1
// (single-CTA allocation).  If racecheck reports the cta_group::2 variant and not the cta_group::1 one,
// the GEMM's report comes from the paired allocation's own shared-memory write (which lands in the slot of
// both CTAs) and not from the GEMM's pipeline.
//   nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o /tmp/rc tools/racecheck_tmem_alloc.cu
//   compute-sanitizer --tool racecheck /tmp/rc 2 ; compute-sanitizer --tool racecheck /tmp/rc 1
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cstdint>

#include "../paper_2507_16099_b200/csrc/ptx.cuh"

using namespace fp8t;

template <int CG>
__global__ void alloc_kernel(uint32_t* out) {
  __shared__ __align__(16) uint32_t slot[4];
  const int warp = threadIdx.x >> 5;
  if (warp == 2) {
    if (CG == 2) {
      tmem_alloc_cg2(smem_u32(slot), 512);
      tmem_relinquish_cg2();
    } else {
      tmem_alloc(smem_u32(slot), 512);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  if (CG == 2) cluster_sync();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot[0];
  if (threadIdx.x == 0) out[blockIdx.x] = base;
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if (CG == 2) tmem_dealloc_cg2(base, 512);
    else tmem_dealloc(base, 512);
  }
}

int main(int argc, char** argv) {
  const int cg = argc > 1 ? atoi(argv[1]) : 2;
  uint32_t* out;
  cudaMalloc(&out, 64 * sizeof(uint32_t));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(8);
  cfg.blockDim = dim3(256);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cg;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cg == 2 ? cudaLaunchKernelEx(&cfg, alloc_kernel<2>, out) : cudaLaunchKernelEx(&cfg, alloc_kernel<1>, out);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  uint32_t h[8];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  printf("cta_group::%d: %s; tmem base of CTA 0..7: %u %u %u %u %u %u %u %u\n", cg, cudaGetErrorString(e), h[0], h[1],
         h[2], h[3], h[4], h[5], h[6], h[7]);
  return e == cudaSuccess ? 0 : 1;
}
