// Internal: fused GEMM -> reduce-scatter over a P2P window (implemented in p2p.cu, used by abi.cpp).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "fp8train.h"
#include "kernels.h"

namespace fp8t {
// Cross-rank barrier on the window (every rank finished reducing the previous epoch, so its staging
// may be overwritten), then fill the problem's rs_* fields: D rows are split into nranks chunks of
// chunk_rows; chunk c goes to rank c's staging slot `rank`.  D must be bf16, chunk_rows % 256 == 0.
fp8_status_t p2p_rs_begin(fp8_p2p_t win, int64_t chunk_rows, int64_t cols, cudaStream_t st, GemmProblem& p);
// Wait for every rank's tiles of this rank's chunk, sum the P staging slots in rank order (fp32) and
// store bf16 [chunk_rows, cols] (row stride ldo elements) to out.
fp8_status_t p2p_rs_end(fp8_p2p_t win, int64_t chunk_rows, int64_t cols, void* out, int64_t ldo, cudaStream_t st);
}  // namespace fp8t
