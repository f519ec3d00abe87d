// Fused FP8 FSDP weight all-gather over NVLink / NVSwitch peer memory (SURVEY §8a row a7,
// PAPER.md:596 enable_fp8_all_gather; reading R-c18: one global scale from the MAX of the shard
// amaxes).  Instead of cast -> ncclAllGather, each rank's cast kernel stores its FP8 codes
// directly into slot `rank` of every rank's gather buffer (peer pointers opened with CUDA IPC),
// so the collective's data movement IS the cast's output stream.
//
// Per call (rank r, epoch e = this window's call counter, identical on all ranks):
//   1. amax(W_r) -> local u32 accumulator                       (existing amax kernel)
//   2. p2p_signal_amax: amax slot r of every peer := (e << 32) | amax   (release, .sys)
//   3. p2p_wait_scale : spin until all P slots carry epoch e; s = fmax / max(max_p amax_p, eps)
//   4. cast_push      : q = satRNE(RN32(W_r * s)) stored to every peer's buffer at slot r;
//                       the last CTA publishes done slot r := e on every peer  (release, .sys)
//   5. p2p_wait_done  : spin until all P done slots >= e  -> the gathered codes are complete
// Step 3 doubles as the cross-rank WAR barrier: rank p pushes epoch-e codes into my buffer only
// after my epoch-e amax signal, which my stream issues after all my earlier work (the GEMMs that
// read epoch e-1's codes).  Every spin has a watchdog (globaltimer, knob watchdog_ms, default 30 s):
// on expiry it writes a fault code to the process-wide fault word (pinned host memory) and gives up
// instead of trapping, so the context survives and the next call returns FP8_ECUDA.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <vector>

#include "comm.h"
#include "fp8train.h"
#include "kernels.h"
#include "p2p_internal.h"
#include "scale.cuh"

namespace fp8t {
fp8_status_t fail(fp8_status_t st, const char* fmt, ...);
fp8_status_t cuda_check(cudaError_t e, const char* what);
fp8_status_t check_fault();

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Watchdog: true (after recording `code` in the fault word) once `timeout_ns` passed since t0.
__device__ __forceinline__ bool watchdog_expired(uint64_t t0, unsigned long long timeout_ns, unsigned* fault,
                                                 unsigned code) {
  if (!timeout_ns || !fault || globaltimer_ns() - t0 <= timeout_ns) return false;
  atomicExch_system(fault, code);
  __threadfence_system();
  return true;
}

__global__ void p2p_signal_amax_kernel(const __grid_constant__ P2PPeers pe, const uint32_t* amax_bits, uint32_t epoch) {
  const unsigned long long v = ((unsigned long long)epoch << 32) | (unsigned long long)*amax_bits;
  for (int p = threadIdx.x; p < pe.P; p += blockDim.x) st_release_sys_u64(&pe.sig[p]->amax[pe.rank], v);
}

template <int FMT>
__global__ void p2p_wait_scale_kernel(P2PSig* mine, int P, uint32_t epoch, float* scale_out, float* amax_out,
                                      unsigned* fault, unsigned long long timeout_ns) {
  const int lane = threadIdx.x;
  uint32_t m = 0;
  const uint64_t t0 = globaltimer_ns();
  for (int p = lane; p < P; p += 32) {
    unsigned long long v;
    while (((v = ld_acquire_sys_u64(&mine->amax[p])) >> 32) != epoch) {
      if (watchdog_expired(t0, timeout_ns, fault, fault_pack(FAULT_P2P_AMAX_WAIT, p, epoch))) break;
      __nanosleep(100);
    }
    m = max(m, (uint32_t)(v & 0xFFFFFFFFull));
  }
  m = __reduce_max_sync(0xffffffffu, m);
  if (lane == 0) {
    const float a = __uint_as_float(m);
    scale_out[0] = scale_of<FMT>(a);
    if (amax_out) amax_out[0] = a;
  }
}

__global__ void p2p_wait_done_kernel(P2PSig* mine, int P, uint32_t epoch, unsigned* fault,
                                     unsigned long long timeout_ns) {
  const uint64_t t0 = globaltimer_ns();
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    while (ld_acquire_sys_u64(&mine->done[p]) < epoch) {
      if (watchdog_expired(t0, timeout_ns, fault, fault_pack(FAULT_P2P_DONE_WAIT, p, epoch))) break;
      __nanosleep(100);
    }
  }
}

// Fused reduce-scatter, owner side (after p2p_wait_done_kernel saw every rank's done[p] >= epoch):
// out = sum_p staging[p] in rank order, fp32, one bf16 rounding.
__global__ void __launch_bounds__(256) p2p_rs_reduce_kernel(const uint4* __restrict__ staging, int P,
                                                            int64_t rows, int64_t cols,
                                                            __nv_bfloat16* __restrict__ out, int64_t ldo) {
  // (the arrival of every rank's tiles was awaited by p2p_wait_done_kernel just before, in stream order)
  const int64_t vec_per_row = cols / 8, n = rows * vec_per_row, slot = rows * vec_per_row;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int p = 0; p < P; ++p) {
      const uint4 v = __ldcg(staging + p * slot + i);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[2 * j] += __uint_as_float(w[j] << 16);
        acc[2 * j + 1] += __uint_as_float(w[j] & 0xFFFF0000u);
      }
    }
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __nv_bfloat162 h = __floats2bfloat162_rn(acc[2 * j], acc[2 * j + 1]);
      o[j] = *reinterpret_cast<uint32_t*>(&h);
    }
    const int64_t r = i / vec_per_row, c = i - r * vec_per_row;
    *reinterpret_cast<uint4*>(out + r * ldo + c * 8) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

}  // namespace fp8t
using namespace fp8t;

#define FP8T_P2P_TRY(expr)               \
  do {                                   \
    fp8_status_t s_ = (expr);            \
    if (s_ != FP8_OK) return s_;         \
  } while (0)

struct fp8_p2p_s {
  int P, rank;
  size_t bytes;            // gather buffer bytes (the window's data part)
  uint8_t* base;           // this rank's window (cudaMalloc), data then P2PSig
  P2PSig* sig;             // this rank's signal block
  P2PPeers peers;
  std::vector<uint8_t*> opened;   // IPC-opened peer bases (to close)
  uint32_t epoch;
  uint8_t** d_bufs = nullptr;      // device copies of peers.buf / peers.sig (read by the GEMM epilogue)
  P2PSig** d_sigs = nullptr;
};

static fp8_status_t upload_tables(fp8_p2p_s* w) {
  const size_t b = sizeof(void*) * (size_t)w->P;
  fp8_status_t s = cuda_check(cudaMalloc(&w->d_bufs, b), "cudaMalloc (peer table)");
  if (s == FP8_OK) s = cuda_check(cudaMalloc(&w->d_sigs, b), "cudaMalloc (peer table)");
  if (s == FP8_OK) s = cuda_check(cudaMemcpy(w->d_bufs, w->peers.buf, b, cudaMemcpyHostToDevice), "cudaMemcpy");
  if (s == FP8_OK) s = cuda_check(cudaMemcpy(w->d_sigs, w->peers.sig, b, cudaMemcpyHostToDevice), "cudaMemcpy");
  return s;
}

static size_t sig_offset(size_t bytes) { return (bytes + 255) & ~size_t(255); }
static size_t window_bytes(size_t bytes) { return sig_offset(bytes) + ((sizeof(P2PSig) + 255) & ~size_t(255)); }

static fp8_status_t alloc_window(size_t bytes, uint8_t** base) {
  fp8_status_t s = cuda_check(cudaMalloc(base, window_bytes(bytes)), "cudaMalloc (p2p window)");
  if (s != FP8_OK) return s;
  return cuda_check(cudaMemset(*base, 0, window_bytes(bytes)), "cudaMemset (p2p window)");
}

extern "C" {

fp8_status_t fp8_p2p_alloc(size_t bytes, int nranks, int rank, fp8_p2p_t* out, uint8_t handle[64]) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t size");
  if (!out || !handle) return fail(FP8_EINVAL, "out/handle: null pointer");
  if (bytes == 0) return fail(FP8_EINVAL, "bytes must be > 0");
  if (nranks < 1 || nranks > P2P_MAXP || rank < 0 || rank >= nranks)
    return fail(FP8_EINVAL, "bad nranks / rank (at most %d ranks)", P2P_MAXP);
  fault_word();   // the watchdog's fault word, allocated at setup (not inside a capture)
  uint8_t* base = nullptr;
  fp8_status_t s = alloc_window(bytes, &base);
  if (s != FP8_OK) return s;
  cudaIpcMemHandle_t h;
  if ((s = cuda_check(cudaIpcGetMemHandle(&h, base), "cudaIpcGetMemHandle")) != FP8_OK) {
    cudaFree(base);
    return s;
  }
  if ((s = cuda_check(cudaDeviceSynchronize(), "sync (window zeroed)")) != FP8_OK) {
    cudaFree(base);
    return s;
  }
  auto* w = new fp8_p2p_s{};
  w->P = nranks;
  w->rank = rank;
  w->bytes = bytes;
  w->base = base;
  w->sig = reinterpret_cast<P2PSig*>(base + sig_offset(bytes));
  w->epoch = 0;
  w->peers.P = nranks;
  w->peers.rank = rank;
  std::memcpy(handle, &h, 64);
  *out = w;
  return FP8_OK;
}

fp8_status_t fp8_p2p_open(fp8_p2p_t w, const uint8_t* handles) {
  if (!w || !handles) return fail(FP8_EINVAL, "win/handles: null pointer");
  if (!w->opened.empty() || w->d_bufs) return fail(FP8_EINVAL, "window already opened");
  fp8_status_t s;
  for (int p = 0; p < w->P; ++p) {
    uint8_t* pb = w->base;
    if (p != w->rank) {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + 64 * (size_t)p, 64);
      void* ptr = nullptr;
      if ((s = cuda_check(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess),
                          "cudaIpcOpenMemHandle (peer window; needs P2P / NVLink)")) != FP8_OK) {
        for (uint8_t* q : w->opened) cudaIpcCloseMemHandle(q);
        w->opened.clear();
        return s;
      }
      pb = static_cast<uint8_t*>(ptr);
      w->opened.push_back(pb);
    }
    w->peers.buf[p] = pb;
    w->peers.sig[p] = reinterpret_cast<P2PSig*>(pb + sig_offset(w->bytes));
  }
  return upload_tables(w);
}

fp8_status_t fp8_p2p_create(fp8_comm_t comm, size_t bytes, fp8_p2p_t* out) {
  if (!comm || !out) return fail(FP8_EINVAL, "comm/out: null pointer");
  if (comm->nranks > P2P_MAXP) return fail(FP8_EUNSUPPORTED, "p2p window: at most %d ranks", P2P_MAXP);
  const int P = comm->nranks, r = comm->rank;
  fp8_p2p_t w = nullptr;
  std::vector<uint8_t> all(64 * (size_t)P);
  fp8_status_t s = fp8_p2p_alloc(bytes, P, r, &w, all.data() + 64 * (size_t)r);
  if (s != FP8_OK) return s;
  // exchange the IPC handles over NCCL (device buffer of P handles, in-place all-gather)
  void* d = nullptr;
  cudaStream_t st = nullptr;
  auto bail = [&](fp8_status_t e) {
    if (d) cudaFree(d);
    if (st) cudaStreamDestroy(st);
    fp8_p2p_destroy(w);
    return e;
  };
  if ((s = cuda_check(cudaMalloc(&d, 64 * (size_t)P), "cudaMalloc")) != FP8_OK) return bail(s);
  if ((s = cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate")) != FP8_OK)
    return bail(s);
  if ((s = cuda_check(cudaMemcpy(static_cast<uint8_t*>(d) + 64 * (size_t)r, all.data() + 64 * (size_t)r, 64,
                                 cudaMemcpyHostToDevice), "cudaMemcpy")) != FP8_OK)
    return bail(s);
  ncclResult_t nr = ncclAllGather(static_cast<uint8_t*>(d) + 64 * (size_t)r, d, 64, ncclUint8, comm->nccl, st);
  if (nr != ncclSuccess) return bail(fail(FP8_ENCCL, "ncclAllGather (ipc handles): %s", ncclGetErrorString(nr)));
  if ((s = cuda_check(cudaStreamSynchronize(st), "sync")) != FP8_OK) return bail(s);
  if ((s = cuda_check(cudaMemcpy(all.data(), d, 64 * (size_t)P, cudaMemcpyDeviceToHost), "cudaMemcpy")) != FP8_OK)
    return bail(s);
  if ((s = fp8_p2p_open(w, all.data())) != FP8_OK) return bail(s);
  // every window is zeroed and mapped before anyone signals into it
  int* one = static_cast<int*>(d);
  nr = ncclAllReduce(one, one, 1, ncclInt32, ncclSum, comm->nccl, st);
  if (nr != ncclSuccess) return bail(fail(FP8_ENCCL, "ncclAllReduce (barrier): %s", ncclGetErrorString(nr)));
  if ((s = cuda_check(cudaStreamSynchronize(st), "sync")) != FP8_OK) return bail(s);
  cudaFree(d);
  cudaStreamDestroy(st);
  *out = w;
  return FP8_OK;
}

fp8_status_t fp8_p2p_create_local(int nranks, size_t bytes, fp8_p2p_t* out) {
  if (!out) return fail(FP8_EINVAL, "out: null pointer");
  if (nranks < 1 || nranks > P2P_MAXP || bytes == 0) return fail(FP8_EINVAL, "bad nranks / bytes");
  fault_word();
  std::vector<uint8_t*> bases(nranks, nullptr);
  for (int p = 0; p < nranks; ++p) {
    fp8_status_t s = alloc_window(bytes, &bases[p]);
    if (s != FP8_OK) {
      for (uint8_t* b : bases)
        if (b) cudaFree(b);
      return s;
    }
  }
  for (int r = 0; r < nranks; ++r) {
    auto* w = new fp8_p2p_s{};
    w->P = nranks;
    w->rank = r;
    w->bytes = bytes;
    w->base = bases[r];
    w->sig = reinterpret_cast<P2PSig*>(bases[r] + sig_offset(bytes));
    w->epoch = 0;
    w->peers.P = nranks;
    w->peers.rank = r;
    for (int p = 0; p < nranks; ++p) {
      w->peers.buf[p] = bases[p];
      w->peers.sig[p] = reinterpret_cast<P2PSig*>(bases[p] + sig_offset(bytes));
    }
    fp8_status_t s = upload_tables(w);
    if (s != FP8_OK) return s;
    out[r] = w;
  }
  return FP8_OK;
}

void* fp8_p2p_buffer(fp8_p2p_t win) { return win ? win->base : nullptr; }

fp8_status_t fp8_p2p_destroy(fp8_p2p_t win) {
  if (!win) return FP8_OK;
  fp8_status_t s = FP8_OK;
  for (uint8_t* p : win->opened)
    if (cudaIpcCloseMemHandle(p) != cudaSuccess) s = fail(FP8_ECUDA, "cudaIpcCloseMemHandle");
  if (cudaFree(win->base) != cudaSuccess) s = fail(FP8_ECUDA, "cudaFree (p2p window)");
  if (win->d_bufs) cudaFree(win->d_bufs);
  if (win->d_sigs) cudaFree(win->d_sigs);
  delete win;
  return s;
}

}  // extern "C"

namespace {

fp8_status_t p2p_check(fp8_p2p_t win, const fp8_hp_t& w, fp8_format_t fmt, const float* amax_in, float* scale_out,
                       float* amax_out) {
  if (!win) return fail(FP8_EINVAL, "win: null");
  FP8T_P2P_TRY(check_fault());
  if (!w.ptr || !scale_out || (!amax_out && !amax_in)) return fail(FP8_EINVAL, "null pointer");
  if (fmt != FP8_E4M3 && fmt != FP8_E5M2) return fail(FP8_EINVAL, "bad fp8 format");
  if (w.dtype != FP8_DT_F32 && w.dtype != FP8_DT_BF16) return fail(FP8_EINVAL, "bad dtype");
  if (w.rows < 16 || w.cols < 16 || w.rows % 16 || w.cols % 16)
    return fail(FP8_EALIGN, "shard rows/cols: multiples of 16");
  if (reinterpret_cast<uintptr_t>(w.ptr) & 15) return fail(FP8_EALIGN, "w_shard must be 16-byte aligned");
  if (w.ld < w.cols || (w.ld * (w.dtype == FP8_DT_F32 ? 4 : 2)) % 16) return fail(FP8_EALIGN, "bad ld");
  if ((size_t)w.rows * (size_t)w.cols * (size_t)win->P > win->bytes)
    return fail(FP8_EINVAL, "window too small for nranks * shard bytes");
  return FP8_OK;
}

// The four phases of one rank's call (see the file header); phase 1 advances the epoch.
fp8_status_t phase_signal(fp8_p2p_t win, const fp8_hp_t& w, const float* amax_in, float* amax_out, cudaStream_t st) {
  const uint32_t epoch = ++win->epoch;
  fp8_status_t s;
  const uint32_t* abits = reinterpret_cast<const uint32_t*>(amax_in);
  if (!amax_in) {
    uint32_t* acc = reinterpret_cast<uint32_t*>(amax_out);
    if ((s = cuda_check(cudaMemsetAsync(acc, 0, 4, st), "memset")) != FP8_OK) return s;
    if ((s = cuda_check(launch_amax(w.ptr, w.dtype == FP8_DT_BF16, w.rows, w.cols, w.ld, 1, acc, nullptr, nullptr, st),
                        "amax")) != FP8_OK)
      return s;
    abits = acc;
  }
  LaunchScope ls(K_SYNC, st);
  p2p_signal_amax_kernel<<<1, 64, 0, st>>>(win->peers, abits, epoch);
  return cuda_check(cudaGetLastError(), "p2p_signal_amax");
}
fp8_status_t phase_wait_scale(fp8_p2p_t win, fp8_format_t fmt, float* scale_out, float* amax_out, cudaStream_t st) {
  LaunchScope ls(K_SYNC, st);
  unsigned* f = fault_word(st);
  const unsigned long long to = watchdog_ns();
  if (fmt == FP8_E4M3) p2p_wait_scale_kernel<0><<<1, 32, 0, st>>>(win->sig, win->P, win->epoch, scale_out, amax_out, f, to);
  else p2p_wait_scale_kernel<1><<<1, 32, 0, st>>>(win->sig, win->P, win->epoch, scale_out, amax_out, f, to);
  return cuda_check(cudaGetLastError(), "p2p_wait_scale");
}
fp8_status_t phase_cast_push(fp8_p2p_t win, const fp8_hp_t& w, fp8_format_t fmt, const float* scale, cudaStream_t st) {
  const size_t chunk = (size_t)w.rows * (size_t)w.cols;
  return cuda_check(launch_cast_push(w.ptr, w.dtype == FP8_DT_BF16, fmt, w.rows, w.cols, w.ld, scale, win->peers,
                                     (int64_t)(chunk * (size_t)win->rank), win->sig, win->epoch, st),
                    "cast_push");
}
fp8_status_t phase_wait_done(fp8_p2p_t win, cudaStream_t st) {
  LaunchScope ls(K_SYNC, st);
  p2p_wait_done_kernel<<<1, 64, 0, st>>>(win->sig, win->P, win->epoch, fault_word(st), watchdog_ns());
  return cuda_check(cudaGetLastError(), "p2p_wait_done");
}

}  // namespace

extern "C" {

fp8_status_t fp8_fsdp_allgather_p2p(fp8_p2p_t win, fp8_hp_t w, fp8_format_t fmt, const float* amax_in,
                                    float* scale_out, float* amax_out, void* stream) {
  FP8T_P2P_TRY(p2p_check(win, w, fmt, amax_in, scale_out, amax_out));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  FP8T_P2P_TRY(phase_signal(win, w, amax_in, amax_out, st));
  FP8T_P2P_TRY(phase_wait_scale(win, fmt, scale_out, amax_out, st));
  FP8T_P2P_TRY(phase_cast_push(win, w, fmt, scale_out, st));
  return phase_wait_done(win, st);
}

fp8_status_t fp8_fsdp_allgather_p2p_local(fp8_p2p_t* wins, int n, const fp8_hp_t* w, fp8_format_t fmt,
                                          const float* const* amax_in, float* const* scale_out,
                                          float* const* amax_out, void* stream) {
  if (!wins || !w || !scale_out || n < 1) return fail(FP8_EINVAL, "null pointer / n < 1");
  for (int r = 0; r < n; ++r) {
    if (!wins[r] || wins[r]->P != n || wins[r]->rank != r) return fail(FP8_EINVAL, "wins must be one local group, in rank order");
    FP8T_P2P_TRY(p2p_check(wins[r], w[r], fmt, amax_in ? amax_in[r] : nullptr, scale_out[r], amax_out ? amax_out[r] : nullptr));
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int r = 0; r < n; ++r) FP8T_P2P_TRY(phase_signal(wins[r], w[r], amax_in ? amax_in[r] : nullptr, amax_out ? amax_out[r] : nullptr, st));
  for (int r = 0; r < n; ++r) FP8T_P2P_TRY(phase_wait_scale(wins[r], fmt, scale_out[r], amax_out ? amax_out[r] : nullptr, st));
  for (int r = 0; r < n; ++r) FP8T_P2P_TRY(phase_cast_push(wins[r], w[r], fmt, scale_out[r], st));
  for (int r = 0; r < n; ++r) FP8T_P2P_TRY(phase_wait_done(wins[r], st));
  return FP8_OK;
}

// ---------------------------------------------------------------------------
// Async-TP FP8 linear forward ("float8 training with async tensor
// parallelism"): sequence-parallel X shards [M_local, K] are all-gathered in FP8 and multiplied by
// this rank's column shard of W [N_local, K] in ONE GEMM launch that overlaps the gather: every rank's
// cast_push stores its codes into slot r of all windows and publishes done[r]; the GEMM's TMA producer
// waits for done[c] before loading chunk c's rows, starting with its own chunk (tile rotation).
//   y [P*M_local, N_local] = X_full W_local^T, tensorwise (global X scale from the signal slots).
// ---------------------------------------------------------------------------
size_t fp8_tp_workspace_bytes(int64_t n_local, int64_t K) { return 1024 + (((size_t)n_local * K + 255) & ~size_t(255)); }

}  // extern "C"

namespace {
struct TpWs {
  float* amax_x; float* scale_x; float* amax_w; float* scale_w; uint8_t* wq;
};
TpWs carve_tp(void* ws) {
  uint8_t* b = static_cast<uint8_t*>(ws);
  return TpWs{reinterpret_cast<float*>(b), reinterpret_cast<float*>(b + 256), reinterpret_cast<float*>(b + 512),
              reinterpret_cast<float*>(b + 768), b + 1024};
}
fp8_status_t tp_check(fp8_p2p_t win, const fp8_linear_cfg_t* cfg, const fp8_hp_t& x, const fp8_hp_t& w, void* y,
                      void* ws, size_t ws_bytes) {
  FP8T_P2P_TRY(check_fault());
  if (!cfg || cfg->recipe != FP8_RECIPE_TENSORWISE) return fail(FP8_EUNSUPPORTED, "async-TP: tensorwise recipe");
  if (cfg->out_dtype != FP8_DT_BF16 && cfg->out_dtype != FP8_DT_F32) return fail(FP8_EINVAL, "bad out_dtype");
  if (!y || !ws || !w.ptr) return fail(FP8_EINVAL, "null pointer");
  if (x.rows % 256) return fail(FP8_EALIGN, "async-TP: M_local must be a multiple of 256");
  if (w.cols != x.cols || w.rows < 16 || w.rows % 16 || w.dtype != x.dtype) return fail(FP8_EINVAL, "w shape / dtype");
  if (w.ld < w.cols || (w.ld * (w.dtype == FP8_DT_F32 ? 4 : 2)) % 16 || (reinterpret_cast<uintptr_t>(w.ptr) & 15))
    return fail(FP8_EALIGN, "w: ld / alignment");
  if ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(ws)) & 255)
    return fail(FP8_EALIGN, "y / ws must be 256-byte aligned");
  if (ws_bytes < fp8_tp_workspace_bytes(w.rows, w.cols)) return fail(FP8_EWORKSPACE, "workspace too small");
  return p2p_check(win, x, (fp8_format_t)cfg->fmt_fwd, nullptr, reinterpret_cast<float*>(ws), reinterpret_cast<float*>(ws));
}
// W cast (local) + the chunk-waiting GEMM of one rank
fp8_status_t tp_gemm(fp8_p2p_t win, const fp8_linear_cfg_t* cfg, const fp8_hp_t& x, const fp8_hp_t& w, void* y,
                     const TpWs& t, cudaStream_t st) {
  const bool wb = w.dtype == FP8_DT_BF16;
  const int ff = cfg->fmt_fwd;
  fp8_status_t s;
  if ((s = cuda_check(cudaMemsetAsync(t.amax_w, 0, 4, st), "memset")) != FP8_OK) return s;
  if ((s = cuda_check(launch_amax(w.ptr, wb, w.rows, w.cols, w.ld, 1, reinterpret_cast<uint32_t*>(t.amax_w), nullptr,
                                  nullptr, st), "amax w")) != FP8_OK)
    return s;
  if ((s = cuda_check(launch_cast(w.ptr, wb, ff, w.rows, w.cols, w.ld, 1, 0, t.amax_w, t.amax_w, t.wq, nullptr,
                                  t.scale_w, nullptr, st), "cast w")) != FP8_OK)
    return s;
  const int64_t M = (int64_t)win->P * x.rows, N = w.rows, K = x.cols;
  GemmProblem p{win->base, t.wq, ff, ff, 0, 0, t.scale_x, t.scale_w, 0, M, N, K, K, K, y,
                cfg->out_dtype == FP8_DT_F32, N};
  p.chunk_done = win->sig->done;
  p.chunk_rows = (int)x.rows;
  p.chunk_epoch = win->epoch;
  p.mrot = win->rank * (int)(x.rows / 256);
  return cuda_check(launch_gemm(p, st), "tp gemm");
}
}  // namespace

extern "C" {

fp8_status_t fp8_tp_allgather_linear_fwd(fp8_p2p_t win, const fp8_linear_cfg_t* cfg, fp8_hp_t x_shard, fp8_hp_t w,
                                         void* y, void* ws, size_t ws_bytes, void* stream) {
  FP8T_P2P_TRY(tp_check(win, cfg, x_shard, w, y, ws, ws_bytes));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const TpWs t = carve_tp(ws);
  const fp8_format_t f = (fp8_format_t)cfg->fmt_fwd;
  FP8T_P2P_TRY(phase_signal(win, x_shard, nullptr, t.amax_x, st));
  FP8T_P2P_TRY(phase_wait_scale(win, f, t.scale_x, t.amax_x, st));
  FP8T_P2P_TRY(phase_cast_push(win, x_shard, f, t.scale_x, st));
  return tp_gemm(win, cfg, x_shard, w, y, t, st);
}

fp8_status_t fp8_tp_allgather_linear_fwd_local(fp8_p2p_t* wins, int n, const fp8_linear_cfg_t* cfg,
                                               const fp8_hp_t* x_shards, const fp8_hp_t* w, void* const* y,
                                               void* const* ws, size_t ws_bytes, void* stream) {
  if (!wins || !x_shards || !w || !y || !ws || n < 1) return fail(FP8_EINVAL, "null pointer / n < 1");
  for (int r = 0; r < n; ++r) {
    if (!wins[r] || wins[r]->P != n || wins[r]->rank != r) return fail(FP8_EINVAL, "wins must be one local group, in rank order");
    FP8T_P2P_TRY(tp_check(wins[r], cfg, x_shards[r], w[r], y[r], ws[r], ws_bytes));
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const fp8_format_t f = (fp8_format_t)cfg->fmt_fwd;
  for (int r = 0; r < n; ++r) FP8T_P2P_TRY(phase_signal(wins[r], x_shards[r], nullptr, carve_tp(ws[r]).amax_x, st));
  for (int r = 0; r < n; ++r) {
    const TpWs t = carve_tp(ws[r]);
    FP8T_P2P_TRY(phase_wait_scale(wins[r], f, t.scale_x, t.amax_x, st));
  }
  for (int r = 0; r < n; ++r) FP8T_P2P_TRY(phase_cast_push(wins[r], x_shards[r], f, carve_tp(ws[r]).scale_x, st));
  for (int r = 0; r < n; ++r) FP8T_P2P_TRY(tp_gemm(wins[r], cfg, x_shards[r], w[r], y[r], carve_tp(ws[r]), st));
  return FP8_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Fused GEMM -> reduce-scatter (used by fp8_linear_bwd_rs, abi.cpp)
// ---------------------------------------------------------------------------
namespace fp8t {

fp8_status_t p2p_rs_begin(fp8_p2p_t win, int64_t chunk_rows, int64_t cols, cudaStream_t st, GemmProblem& p) {
  if (!win) return fail(FP8_EINVAL, "rs window: null");
  if (chunk_rows <= 0 || chunk_rows % 256 || cols % 16) return fail(FP8_EALIGN, "reduce-scatter: chunk rows % 256, cols % 16");
  if ((size_t)win->P * (size_t)chunk_rows * (size_t)cols * 2 > win->bytes)
    return fail(FP8_EINVAL, "rs window too small (needs nranks * chunk_rows * cols * 2 bytes)");
  // barrier: every rank reached this call after its previous reduce (stream order), so no staging
  // slot of the previous epoch is still being read when this epoch's tiles land
  fp8_hp_t dummy{win->base, FP8_DT_BF16, 16, 16, 16};
  FP8T_P2P_TRY(phase_signal(win, dummy, win->sig->scratch, nullptr, st));
  FP8T_P2P_TRY(phase_wait_scale(win, FP8_E4M3, win->sig->scratch + 1, win->sig->scratch + 2, st));
  p.rs_bufs = win->d_bufs;
  p.rs_sigs = win->d_sigs;
  p.rs_cnt = win->sig->rs_cnt;
  p.rs_rank = win->rank;
  p.rs_chunk_rows = (int)chunk_rows;
  p.rs_epoch = win->epoch;
  p.ldd = cols;
  return FP8_OK;
}

fp8_status_t p2p_rs_end(fp8_p2p_t win, int64_t chunk_rows, int64_t cols, void* out, int64_t ldo, cudaStream_t st) {
  FP8T_P2P_TRY(phase_wait_done(win, st));   // one spinning warp; the reduce below never spins
  const int64_t n = chunk_rows * cols / 8;
  int64_t g = (n + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  LaunchScope ls(K_SYNC, st);
  p2p_rs_reduce_kernel<<<(unsigned)g, 256, 0, st>>>(reinterpret_cast<const uint4*>(win->base), win->P, chunk_rows, cols,
                                                    static_cast<__nv_bfloat16*>(out), ldo);
  return cuda_check(cudaGetLastError(), "rs reduce");
}

}  // namespace fp8t


// ---------------------------------------------------------------------------
// Async-TP FP8 linear backward (pairs with fp8_tp_allgather_linear_fwd): the row-parallel dX
// partials are reduce-scattered to the token shards inside the GEMM (fused RS epilogue), dW_r is
// local.  Per rank r:  dY_r [M, N_local] tensorwise cast (local scale) ->
//   dX partial = dYq W_r (contraction over N_local) -> rows of token chunk c stored into rank c's
//                staging (rs_win), summed there in rank order  -> dx_shard [M_local, K]
//   dW_r       = dYq^T X_full (the FP8 codes gathered by the forward, still in win)
// both problems in one persistent launch.
// ---------------------------------------------------------------------------
extern "C" {

size_t fp8_tp_bwd_workspace_bytes(int64_t M, int64_t n_local) { return 1024 + (((size_t)M * n_local + 255) & ~size_t(255)); }

fp8_status_t fp8_tp_linear_bwd(fp8_p2p_t win, const void* fwd_ws, fp8_p2p_t rs_win, const fp8_linear_cfg_t* cfg,
                               fp8_hp_t dy, int64_t K, void* dx_shard, void* dw, void* ws, size_t ws_bytes,
                               void* stream) {
  FP8T_P2P_TRY(check_fault());
  if (!win || !rs_win || !fwd_ws || !cfg || !ws || !dx_shard || !dw) return fail(FP8_EINVAL, "null pointer");
  if (cfg->recipe != FP8_RECIPE_TENSORWISE || cfg->out_dtype != FP8_DT_BF16)
    return fail(FP8_EUNSUPPORTED, "async-TP backward: tensorwise recipe, bf16 outputs");
  if (win->P != rs_win->P || win->rank != rs_win->rank) return fail(FP8_EINVAL, "win / rs_win: different groups");
  const int64_t M = dy.rows, Nl = dy.cols, Ml = M / win->P;
  if (M % ((int64_t)win->P * 256) || Nl % 16 || K % 16 || dy.ld < Nl) return fail(FP8_EALIGN, "shapes: M % (256 P), N, K % 16");
  if ((size_t)M * K > win->bytes) return fail(FP8_EINVAL, "win does not hold the forward's gathered X");
  if (ws_bytes < fp8_tp_bwd_workspace_bytes(M, Nl)) return fail(FP8_EWORKSPACE, "workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const TpWs t = carve_tp(const_cast<void*>(fwd_ws));
  uint8_t* b = static_cast<uint8_t*>(ws);
  float* amax_g = reinterpret_cast<float*>(b);
  float* scale_g = reinterpret_cast<float*>(b + 256);
  uint8_t* gq = b + 1024;
  const bool gb = dy.dtype == FP8_DT_BF16;
  const int ff = cfg->fmt_fwd, fg = cfg->fmt_grad;
  fp8_status_t s;
  if ((s = cuda_check(cudaMemsetAsync(amax_g, 0, 4, st), "memset")) != FP8_OK) return s;
  if ((s = cuda_check(launch_amax(dy.ptr, gb, M, Nl, dy.ld, 1, reinterpret_cast<uint32_t*>(amax_g), nullptr, nullptr, st),
                      "amax dy")) != FP8_OK)
    return s;
  if ((s = cuda_check(launch_cast(dy.ptr, gb, fg, M, Nl, dy.ld, 1, 0, amax_g, amax_g, gq, nullptr, scale_g, nullptr, st),
                      "cast dy")) != FP8_OK)
    return s;
  GemmProblem ps[2];
  // dW_r [Nl, K] = dY^T X_full: both MN-major (contraction over the M tokens)
  ps[0] = GemmProblem{gq, win->base, fg, ff, 1, 1, scale_g, t.scale_x, 0, Nl, K, M, Nl, K, dw, 0, K};
  // dX partial [M, K] = dY W_r: A K-major over Nl, B = W_r codes [Nl, K] read MN-major; reduce-scattered
  ps[1] = GemmProblem{gq, t.wq, fg, ff, 0, 1, scale_g, t.scale_w, 0, M, K, Nl, Nl, K, dx_shard, 0, K};
  FP8T_P2P_TRY(p2p_rs_begin(rs_win, Ml, K, st, ps[1]));
  if ((s = cuda_check(launch_gemms(ps, 2, st), "tp bwd gemms")) != FP8_OK) return s;
  return p2p_rs_end(rs_win, Ml, K, dx_shard, K, st);
}

}  // extern "C"
