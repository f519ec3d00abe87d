// FSDP2-style FP8 weight all-gather over NCCL (NVLink 5 / NVSwitch on B200).
//
// PAPER.md:596 (Appendix A, tensorwise): "enable_fp8_all_gather which will perform the
// all-gathers in FSDP using FP8 to reduce communication overhead".  Reading R-c18: one
// global scale per weight from the all-reduced MAX of the per-shard amaxes, so the
// gathered bytes equal the unsharded tensorwise cast on every rank.
//
// Step per rank:  amax(W_r) -> ncclAllReduce(MAX) -> cast W_r into slot r of w_full with
// s = RN32(fmax/max(amax,eps)) -> in-place ncclAllGather of the FP8 bytes.  The amax is
// reduced as its u32 bit pattern: for non-negative floats u32 order == float order, so
// the MAX is exact and needs no float NaN semantics.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>

#include "fp8train.h"
#include "kernels.h"

namespace fp8t {
fp8_status_t fail(fp8_status_t st, const char* fmt, ...);
fp8_status_t cuda_check(cudaError_t e, const char* what);
}  // namespace fp8t
using namespace fp8t;

struct fp8_comm_s {
  ncclComm_t nccl;
  int nranks, rank;
};

static fp8_status_t nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return FP8_OK;
  return fail(FP8_ENCCL, "%s: %s", what, ncclGetErrorString(r));
}

extern "C" {

fp8_status_t fp8_comm_get_unique_id(uint8_t id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  if (!id) return fail(FP8_EINVAL, "id: null pointer");
  ncclUniqueId u;
  fp8_status_t s = nccl_check(ncclGetUniqueId(&u), "ncclGetUniqueId");
  if (s != FP8_OK) return s;
  std::memcpy(id, &u, 128);
  return FP8_OK;
}

fp8_status_t fp8_comm_init(fp8_comm_t* comm, const uint8_t id[128], int nranks, int rank) {
  if (!comm || !id) return fail(FP8_EINVAL, "comm/id: null pointer");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(FP8_EINVAL, "bad nranks/rank");
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t c;
  fp8_status_t s = nccl_check(ncclCommInitRank(&c, nranks, u, rank), "ncclCommInitRank");
  if (s != FP8_OK) return s;
  *comm = new fp8_comm_s{c, nranks, rank};
  return FP8_OK;
}

fp8_status_t fp8_comm_destroy(fp8_comm_t comm) {
  if (!comm) return FP8_OK;
  fp8_status_t s = nccl_check(ncclCommDestroy(comm->nccl), "ncclCommDestroy");
  delete comm;
  return s;
}

size_t fp8_fsdp_workspace_bytes(fp8_hp_t) { return 0; }

fp8_status_t fp8_fsdp_precompute_amax(fp8_comm_t comm, const fp8_hp_t* w, int n, float* amax_out, void* stream) {
  if (!comm) return fail(FP8_EINVAL, "comm: null");
  fp8_status_t s = fp8_amax_multi(w, n, amax_out, stream);
  if (s != FP8_OK) return s;
  return nccl_check(ncclAllReduce(amax_out, amax_out, (size_t)n, ncclUint32, ncclMax, comm->nccl,
                                  static_cast<cudaStream_t>(stream)),
                    "ncclAllReduce");
}

fp8_status_t fp8_fsdp_allgather(fp8_comm_t comm, fp8_hp_t w, fp8_format_t fmt, uint8_t* w_full, float* scale_out,
                                float* amax_out, void* ws, size_t ws_bytes, void* stream) {
  return fp8_fsdp_allgather_ex(comm, w, fmt, nullptr, w_full, scale_out, amax_out, ws, ws_bytes, stream);
}

fp8_status_t fp8_fsdp_allgather_ex(fp8_comm_t comm, fp8_hp_t w, fp8_format_t fmt, const float* amax_in,
                                   uint8_t* w_full, float* scale_out, float* amax_out, void*, size_t, void* stream) {
  if (!comm) return fail(FP8_EINVAL, "comm: null");
  if (!w.ptr || !w_full || !scale_out || (!amax_out && !amax_in)) return fail(FP8_EINVAL, "null pointer");
  if (fmt != FP8_E4M3 && fmt != FP8_E5M2) return fail(FP8_EINVAL, "bad fp8 format");
  if (w.dtype != FP8_DT_F32 && w.dtype != FP8_DT_BF16) return fail(FP8_EINVAL, "bad dtype");
  if (w.rows < 16 || w.cols < 16 || w.rows % 16 || w.cols % 16) return fail(FP8_EALIGN, "shard rows/cols: multiples of 16");
  if ((reinterpret_cast<uintptr_t>(w.ptr) | reinterpret_cast<uintptr_t>(w_full)) & 15)
    return fail(FP8_EALIGN, "pointers must be 16-byte aligned");
  if (w.ld < w.cols || (w.ld * (w.dtype == FP8_DT_F32 ? 4 : 2)) % 16) return fail(FP8_EALIGN, "bad ld");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool bf16 = w.dtype == FP8_DT_BF16;
  const size_t chunk = (size_t)w.rows * (size_t)w.cols;
  uint8_t* slot = w_full + (size_t)comm->rank * chunk;
  fp8_status_t s;
  if (!amax_in) {
    uint32_t* acc = reinterpret_cast<uint32_t*>(amax_out);
    if ((s = cuda_check(cudaMemsetAsync(acc, 0, 4, st), "memset")) != FP8_OK) return s;
    if ((s = cuda_check(launch_amax(w.ptr, bf16, w.rows, w.cols, w.ld, 1, acc, nullptr, nullptr, st), "amax")) !=
        FP8_OK)
      return s;
    if ((s = nccl_check(ncclAllReduce(acc, acc, 1, ncclUint32, ncclMax, comm->nccl, st), "ncclAllReduce")) != FP8_OK)
      return s;
    amax_in = amax_out;
  }
  if ((s = cuda_check(launch_cast(w.ptr, bf16, fmt, w.rows, w.cols, w.ld, 1, 0, amax_in, amax_in, slot, nullptr,
                                  scale_out, nullptr, st),
                      "cast")) != FP8_OK)
    return s;
  return nccl_check(ncclAllGather(slot, w_full, chunk, ncclUint8, comm->nccl, st), "ncclAllGather");
}

}  // extern "C"
