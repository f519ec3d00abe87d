// Scale rule of the tensorwise / rowwise recipes, shared by the cast and the P2P gather kernels.
#pragma once
#include <cuda_runtime.h>

namespace fp8t {

// eps = fp32(1e-12) (DESIGN.md R-c5), written as its bit pattern.
__device__ __forceinline__ float kEps() { return __int_as_float(0x2B8CBCCC); }
template <int FMT> __device__ __forceinline__ float kFmax() { return FMT == 0 ? 448.0f : 57344.0f; }
template <int FMT> __device__ __forceinline__ int kEmax() { return FMT == 0 ? 8 : 15; }

// s = RN32(fmax / max(amax, eps)), IEEE division (R-c3, R-c6).
template <int FMT>
__device__ __forceinline__ float scale_of(float amax) {
  return __fdiv_rn(kFmax<FMT>(), fmaxf(amax, kEps()));
}

}  // namespace fp8t
