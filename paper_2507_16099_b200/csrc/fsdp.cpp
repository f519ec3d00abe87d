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
#include "comm.h"
#include "kernels.h"

namespace fp8t {
fp8_status_t fail(fp8_status_t st, const char* fmt, ...);
fp8_status_t cuda_check(cudaError_t e, const char* what);
fp8_status_t check_fault();
}  // namespace fp8t
using namespace fp8t;


static fp8_status_t nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return FP8_OK;
  return fail(FP8_ENCCL, "%s: %s", what, ncclGetErrorString(r));
}

// Health of a communicator before enqueuing more work on it: an asynchronous NCCL error (a peer died,
// a network / NVLink fault, a timed-out operation) is polled with ncclCommGetAsyncError and
// returned as FP8_ENCCL, as is an earlier device fault recorded in the fault word.
static fp8_status_t comm_health(fp8_comm_t comm) {
  if (!comm) return fail(FP8_EINVAL, "comm: null");
  fp8_status_t s = check_fault();
  if (s != FP8_OK) return s;
  ncclResult_t ae = ncclSuccess;
  ncclResult_t r = ncclCommGetAsyncError(comm->nccl, &ae);
  if (r != ncclSuccess) return fail(FP8_ENCCL, "ncclCommGetAsyncError: %s", ncclGetErrorString(r));
  if (ae != ncclSuccess && ae != ncclInProgress)
    return fail(FP8_ENCCL, "communicator in error state (asynchronous NCCL error): %s", ncclGetErrorString(ae));
  return FP8_OK;
}

extern "C" {

fp8_status_t fp8_comm_check(fp8_comm_t comm) { return comm_health(comm); }

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
  {
    const fp8_status_t h = comm_health(comm);
    if (h != FP8_OK) return h;
  }
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
  {
    const fp8_status_t h = comm_health(comm);
    if (h != FP8_OK) return h;
  }
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

// ---------------------------------------------------------------------------
// MXFP8 FSDP gather.  A 32-block never crosses a shard boundary when
// rows_local % 128 == 0, so every E8M0 code is shard-local: no amax exchange.  Rank r casts its
// shard straight into its slots (dim0 codes + blocked scales are contiguous per shard; dim1 codes
// too, in the row-major MX32_RM layout), the dim1 scales into slot r of a rank-major staging
// buffer; one NCCL group all-gathers the four buffers; the dim1 scales are then re-tiled into
// the full blocked layout.
// ---------------------------------------------------------------------------
size_t fp8_fsdp_mx_workspace_bytes(fp8_hp_t w, int nranks) {
  return nranks > 0 && w.rows > 0 && w.cols > 0 ? (size_t)nranks * (size_t)w.rows * (size_t)w.cols / 32 : 0;
}

fp8_status_t fp8_mx_scales_unshard(const uint8_t* rank_major, int nranks, int64_t rows_local, int64_t cols,
                                   uint8_t* out, void* stream) {
  if (!rank_major || !out) return fail(FP8_EINVAL, "null pointer");
  if (nranks < 1 || rows_local < 128 || cols < 128 || rows_local % 128 || cols % 128)
    return fail(FP8_EALIGN, "rows_local and cols must be positive multiples of 128");
  if ((reinterpret_cast<uintptr_t>(rank_major) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(FP8_EALIGN, "pointers must be 16-byte aligned");
  return cuda_check(launch_sf_unshard(rank_major, nranks, cols / 128, rows_local / 128, out,
                                      static_cast<cudaStream_t>(stream)),
                    "sf_unshard");
}

fp8_status_t fp8_fsdp_allgather_mx(fp8_comm_t comm, fp8_hp_t w, fp8_mx_round_t mx_round, fp8_tensor_t* out, void* ws,
                                   size_t ws_bytes, void* stream) {
  if (!comm) return fail(FP8_EINVAL, "comm: null");
  if (!w.ptr || !out || !out->q || !out->scale) return fail(FP8_EINVAL, "null pointer (w, out, out->q, out->scale)");
  if (out->fmt != FP8_E4M3 && out->fmt != FP8_E5M2) return fail(FP8_EINVAL, "bad fp8 format");
  if (out->gran != FP8_GRAN_MX32_RM) return fail(FP8_EUNSUPPORTED, "out->gran must be FP8_GRAN_MX32_RM");
  if (mx_round != FP8_MX_FLOOR && mx_round != FP8_MX_RCEIL) return fail(FP8_EINVAL, "bad mx_round");
  if (w.dtype != FP8_DT_F32 && w.dtype != FP8_DT_BF16) return fail(FP8_EINVAL, "bad dtype");
  if ((out->q_t == nullptr) != (out->scale_t == nullptr)) return fail(FP8_EINVAL, "q_t and scale_t: both or neither");
  if (w.rows < 128 || w.cols < 128 || w.rows % 128 || w.cols % 128)
    return fail(FP8_EALIGN, "MX shard rows/cols: multiples of 128");
  if (out->rows != (int64_t)comm->nranks * w.rows || out->cols != w.cols) return fail(FP8_EINVAL, "out shape");
  if (w.ld < w.cols || (w.ld * (w.dtype == FP8_DT_F32 ? 4 : 2)) % 16) return fail(FP8_EALIGN, "bad ld");
  uintptr_t al = reinterpret_cast<uintptr_t>(w.ptr) | reinterpret_cast<uintptr_t>(out->q) |
                 reinterpret_cast<uintptr_t>(out->scale) | reinterpret_cast<uintptr_t>(out->q_t) |
                 reinterpret_cast<uintptr_t>(out->scale_t) | reinterpret_cast<uintptr_t>(ws);
  if (al & 15) return fail(FP8_EALIGN, "pointers must be 16-byte aligned");
  const bool dim1 = out->q_t != nullptr;
  if (dim1 && (!ws || ws_bytes < fp8_fsdp_mx_workspace_bytes(w, comm->nranks)))
    return fail(FP8_EWORKSPACE, "workspace too small");
  {
    const fp8_status_t h = comm_health(comm);
    if (h != FP8_OK) return h;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t chunk = (size_t)w.rows * (size_t)w.cols, r = (size_t)comm->rank;
  uint8_t* q0 = out->q + r * chunk;
  uint8_t* s0 = static_cast<uint8_t*>(out->scale) + r * chunk / 32;
  uint8_t* q1 = dim1 ? out->q_t + r * chunk : nullptr;
  uint8_t* s1 = dim1 ? static_cast<uint8_t*>(ws) + r * chunk / 32 : nullptr;
  fp8_status_t s;
  if ((s = cuda_check(launch_mx_cast(w.ptr, w.dtype == FP8_DT_BF16, out->fmt, mx_round == FP8_MX_RCEIL, w.rows,
                                     w.cols, w.ld, q0, s0, q1, s1, st, false),
                      "mx cast")) != FP8_OK)
    return s;
  if ((s = nccl_check(ncclGroupStart(), "ncclGroupStart")) != FP8_OK) return s;
  ncclResult_t e = ncclAllGather(q0, out->q, chunk, ncclUint8, comm->nccl, st);
  if (e == ncclSuccess) e = ncclAllGather(s0, out->scale, chunk / 32, ncclUint8, comm->nccl, st);
  if (e == ncclSuccess && dim1) e = ncclAllGather(q1, out->q_t, chunk, ncclUint8, comm->nccl, st);
  if (e == ncclSuccess && dim1) e = ncclAllGather(s1, ws, chunk / 32, ncclUint8, comm->nccl, st);
  ncclResult_t e2 = ncclGroupEnd();
  if ((s = nccl_check(e != ncclSuccess ? e : e2, "ncclAllGather (mx group)")) != FP8_OK) return s;
  if (!dim1) return FP8_OK;
  return fp8_mx_scales_unshard(static_cast<const uint8_t*>(ws), comm->nranks, w.rows, w.cols,
                               static_cast<uint8_t*>(out->scale_t), stream);
}

}  // extern "C"
