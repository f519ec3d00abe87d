// TMA L2 -> SMEM throughput ceiling on this part: every CTA keeps S box loads (16 KB each) in flight into a
// smem ring and re-issues each as soon as it lands, cycling over its own slice of a buffer that is either
// L2-resident (MB <= ~96) or not (MB >= 1024).  No consumer: the aggregate bytes / time is the ceiling the
// GEMM's operand stream and the cast kernels' tile reads can approach.  The buffer is a 2-D
// tensor with rows of `pitch` bytes and the box is `inner` bytes x (16384 / inner) rows (inner 128 with
// SWIZZLE_128B = the GEMM's operand box; inner 256 / 512 with no swizzle = the cast kernels' bf16 tiles).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda -o /tmp/tma_bw tools/tma_bw.cu
//   /tmp/tma_bw <buffer MB> <CTAs per SM> <stages> [pitch bytes = 128] [inner bytes = 128]
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

#include "../paper_2507_16099_b200/csrc/ptx.cuh"

using namespace fp8t;

__global__ void tma_bw_kernel(const __grid_constant__ CUtensorMap m, int rows_total, int iters, int S,
                              unsigned long long* sink, int box_rows, int col_boxes) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  const uint32_t bars = base + S * 16384;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) mbar_init(bars + 8 * s, 1);
  fence_mbar_init();
  const int boxes = (rows_total / box_rows) * col_boxes;   // boxes in the buffer, row-major over the box grid
  int next = (blockIdx.x * 7919) % boxes;
  const int inner = 16384 / box_rows;
  auto issue = [&](int s) {
    mbar_arrive_expect_tx(bars + 8 * s, 16384);
    tma_load_2d(base + s * 16384, &m, (next % col_boxes) * inner, (next / col_boxes) * box_rows, bars + 8 * s, 0);
    next += gridDim.x;
    if (next >= boxes) next -= boxes;
  };
  for (int s = 0; s < S; ++s) issue(s);
  uint32_t phase = 0;
  for (int it = 0; it < iters; ++it) {
    for (int s = 0; s < S; ++s) {
      mbar_wait(bars + 8 * s, phase);
      issue(s);
    }
    phase ^= 1;
  }
  for (int s = 0; s < S; ++s) mbar_wait(bars + 8 * s, phase);
  if (blockIdx.x == 0) *sink = next;
}

int main(int argc, char** argv) {
  const int mb = argc > 1 ? atoi(argv[1]) : 64;
  const int per_sm = argc > 2 ? atoi(argv[2]) : 1;
  const int S = argc > 3 ? atoi(argv[3]) : 8;
  const int pitch = argc > 4 ? atoi(argv[4]) : 128;
  const int inner = argc > 5 ? atoi(argv[5]) : 128;
  const int box_rows = 16384 / inner;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = (size_t)mb << 20;
  uint8_t* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const int rows = (int)(bytes / pitch);
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)pitch, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)pitch};
  cuuint32_t box[2] = {(cuuint32_t)inner, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   inner == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("{\"err\": \"tensor map %d\"}\n", (int)r); return 1; }
  const int smem = S * 16384 + 8 * S + 1024;
  cudaFuncSetAttribute(tma_bw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = nsm * per_sm, iters = 400;
  const int col_boxes = pitch / inner;
  tma_bw_kernel<<<grid, 32, smem>>>(m, rows, 20, S, sink, box_rows, col_boxes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  tma_bw_kernel<<<grid, 32, smem>>>(m, rows, iters, S, sink, box_rows, col_boxes);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double moved = (double)grid * (iters + 1) * S * 16384.0;
  printf("{\"buffer_MB\": %d, \"ctas_per_sm\": %d, \"stages\": %d, \"pitch\": %d, \"inner\": %d, \"TBps\": %.2f, "
         "\"err\": \"%s\"}\n", mb, per_sm, S, pitch, inner, moved / (ms * 1e-3) / 1e12, cudaGetErrorString(e));
  return 0;
}
