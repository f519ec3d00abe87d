// C-ABI implementation (include/fp8train.h): validation, workspace carving and the
// per-recipe orchestration of the Float8Linear forward/backward (Appendix A,
// PAPER.md:594-598).  Every compute step runs in the kernels of cast_kernels.cu /
// gemm_kernels.cu; this file only checks arguments and enqueues work.
#include "fp8train.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.h"
#include "p2p_internal.h"

namespace fp8t {

static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// ---- kernel-variant knobs (defaults = the product path) ----
struct KnobDef { const char* name; int def, lo, hi; };
static const KnobDef kKnobs[KNOB_COUNT] = {
    {"amax_tile_tma", 1, 0, 1},     {"cast_grid", 0, 0, 1 << 20},  {"amax_blocks_per_sm", 8, 1, 9},
    {"amax_loads", 8, 4, 16},       {"mx_cast_tma", 1, 0, 1},      {"gemm_cta_group", 2, 1, 2},
    {"gemm_debug", 0, 0, 1 << 16},  {"gemm_sched", 1, 0, 1},       {"mx_sf_split", 1, 0, 8},
    {"gemm_raster", -1, -1, 64},    {"mx_n192", 0, 0, 1},          {"gemm_stages", 3, 3, 6},
    {"gemm_epi", 0, 0, 8},          {"mx_transposed", 0, 0, 1},    {"tw_dual", 1, 0, 1},
    {"gemm_kserp", 1, 0, 1},        {"gemm_n512", 2, 0, 2},        {"gemm_l2pf", 0, 0, 64},
    {"mx_cast_occ3", 0, 0, 1},      {"amax_bulk", 1, 0, 1},        {"amax_rc", 1, 0, 1},
    {"amax_rc_debug", 0, 0, 1},     {"group_batch", 1, 0, 1},
    {"mx_cast_debug", 0, 0, 1},     {"mx_cast_ws", 0, 0, 1},        {"gemm_st_ef", 0, 0, 1},
    {"wait_sleep", 0, 0, 15},       {"gemm_l2hint", 0, 0, 3},       {"gemm_afill", 0, 0, 1},        {"mx_cast_tstore", 1, 0, 1},     {"cast_rc_tma", 1, 0, 2},        {"cast_rc_wide", 0, 0, 1},       {"gemm_epi_tma", 0, 0, 1},
    {"watchdog_ms", 30000, 0, 1 << 30},
};
static std::atomic<int> g_knobs[KNOB_COUNT];
// defaults come from the table (one source of truth); a table shorter than the enum leaves a null name
static const bool g_knobs_ready = [] {
  for (int i = 0; i < KNOB_COUNT; ++i) {
    if (!kKnobs[i].name) {
      std::fprintf(stderr, "fp8train: knob table incomplete (entry %d)\n", i);
      std::abort();
    }
    g_knobs[i].store(kKnobs[i].def, std::memory_order_relaxed);
  }
  return true;
}();
int knob(Knob k) { return g_knobs[k].load(std::memory_order_relaxed); }
static int knob_index(const char* name) {
  if (!name) return -1;
  for (int i = 0; i < KNOB_COUNT; ++i)
    if (std::strcmp(name, kKnobs[i].name) == 0) return i;
  return -1;
}

// ---- asynchronous device faults ----
fp8_status_t fail(fp8_status_t st, const char* fmt, ...);
static std::mutex g_fault_mu;
static std::atomic<unsigned*> g_fault_dev{nullptr};
static volatile unsigned* g_fault_host = nullptr;
static bool g_fault_tried = false;
unsigned* fault_word(cudaStream_t st) {
  unsigned* d = g_fault_dev.load(std::memory_order_acquire);
  if (d) return d;
  // allocate lazily, but never while `st` is being captured into a CUDA graph (cudaHostAlloc is not a
  // stream operation and would invalidate the capture): such a launch runs without fault reporting
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (st && (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)) return nullptr;
  std::lock_guard<std::mutex> lk(g_fault_mu);
  if (g_fault_tried) return g_fault_dev.load();
  g_fault_tried = true;
  void* h = nullptr;
  if (cudaHostAlloc(&h, 64, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  std::memset(h, 0, 64);
  void* dp = nullptr;
  if (cudaHostGetDevicePointer(&dp, h, 0) != cudaSuccess) {
    cudaGetLastError();
    cudaFreeHost(h);
    return nullptr;
  }
  g_fault_host = static_cast<volatile unsigned*>(h);
  g_fault_dev.store(static_cast<unsigned*>(dp), std::memory_order_release);
  return static_cast<unsigned*>(dp);
}
unsigned long long watchdog_ns() { return (unsigned long long)knob(KNOB_WATCHDOG_MS) * 1000000ull; }
fp8_status_t check_fault() {
  if (!g_fault_host) return FP8_OK;
  const unsigned f = *g_fault_host;
  if (!f) return FP8_OK;
  *g_fault_host = 0;
  const unsigned code = f >> 24, peer = (f >> 16) & 0xFF, ep = f & 0xFFFF;
  switch (code) {
    case FAULT_P2P_AMAX_WAIT:
      return fail(FP8_ECUDA, "earlier P2P gather: rank %u's amax signal (epoch %u) never arrived within the "
                  "watchdog; its outputs are invalid", peer, ep);
    case FAULT_P2P_DONE_WAIT:
      return fail(FP8_ECUDA, "earlier P2P call: rank %u's pushes / tiles (epoch %u) never completed within the "
                  "watchdog; its outputs are invalid", peer, ep);
    case FAULT_TP_CHUNK_WAIT:
      return fail(FP8_ECUDA, "earlier async-TP GEMM: A chunk %u never arrived within the watchdog; its outputs "
                  "are invalid", peer);
    case FAULT_GROUP_OFFSETS:
      return fail(FP8_EINVAL, "earlier grouped GEMM: device group offsets invalid (need 0 = offs[0] <= ... <= "
                  "offs[G] = extent, multiples of 128); its outputs are invalid");
    default:
      return fail(FP8_ECUDA, "earlier kernel reported device fault 0x%08x", f);
  }
}

// ---- per-device host caches ----
cudaError_t current_device(int* dev) {
  cudaError_t e = cudaGetDevice(dev);
  if (e == cudaSuccess && *dev < 0) return cudaErrorInvalidDevice;
  return e;
}
int device_sm_count() {
  static std::atomic<int> cache[MAX_DEVICES];
  int dev = 0;
  if (current_device(&dev) != cudaSuccess) return 148;
  int n = dev < MAX_DEVICES ? cache[dev].load(std::memory_order_relaxed) : 0;
  if (n > 0) return n;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  if (dev < MAX_DEVICES) cache[dev].store(n, std::memory_order_relaxed);
  return n;
}

// ---- optional per-launch event timing (fp8_profile_enable / fp8_profile_collect) ----
struct ProfRec { int kind; cudaEvent_t a, b; };
static std::atomic<int> g_prof_on{0};
static std::mutex g_prof_mu;
static std::vector<ProfRec> g_prof;          // recorded, not yet collected
static std::vector<cudaEvent_t> g_prof_free;  // event pool

static cudaEvent_t prof_event() {
  if (!g_prof_free.empty()) {
    cudaEvent_t e = g_prof_free.back();
    g_prof_free.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

LaunchScope::LaunchScope(int kind, cudaStream_t s) : slot(-1), st(s) {
  if (!g_prof_on.load(std::memory_order_relaxed)) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  ProfRec r{kind, prof_event(), prof_event()};
  cudaEventRecord(r.a, s);
  g_prof.push_back(r);
  slot = (int)g_prof.size() - 1;
}
LaunchScope::~LaunchScope() {
  count_launch();
  if (slot < 0) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (slot < (int)g_prof.size()) cudaEventRecord(g_prof[slot].b, st);
}

static thread_local std::string g_err;

fp8_status_t fail(fp8_status_t st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

fp8_status_t cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return FP8_OK;
  return fail(FP8_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define FP8T_TRY(expr)                         \
  do {                                         \
    fp8_status_t _s = (expr);                  \
    if (_s != FP8_OK) return _s;               \
  } while (0)
#define FP8T_CUDA(expr, what) FP8T_TRY(cuda_check((expr), (what)))

static inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
static inline size_t al(size_t b) { return (b + 255) & ~size_t(255); }
static inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
static inline size_t esize(fp8_dtype_t d) { return d == FP8_DT_F32 ? 4 : 2; }
// MXFP8 linear: dim1 codes written transposed and read K-major (knob mx_transposed = 1, the A/B
// variant) instead of row-major and read MN-major (default).  Forward and backward must agree.
static inline bool mx_transposed() { return knob(KNOB_MX_TRANSPOSED) == 1; }

static fp8_status_t check_hp(const fp8_hp_t& x, const char* name, bool need_ptr = true) {
  if (x.dtype != FP8_DT_F32 && x.dtype != FP8_DT_BF16) return fail(FP8_EINVAL, "%s: bad dtype", name);
  if (x.rows < 16 || x.cols < 16) return fail(FP8_EINVAL, "%s: rows/cols must be >= 16", name);
  if (x.rows % 16 || x.cols % 16) return fail(FP8_EALIGN, "%s: rows and cols must be multiples of 16", name);
  if (x.ld < x.cols) return fail(FP8_EINVAL, "%s: ld < cols", name);
  if ((x.ld * (int64_t)esize(x.dtype)) % 16) return fail(FP8_EALIGN, "%s: ld*elem_size must be a multiple of 16", name);
  if (x.rows > (int64_t)1 << 31 || x.cols > (int64_t)1 << 31) return fail(FP8_EINVAL, "%s: dims too large", name);
  // the tile casts address the rows of a 128-row tile by 32-bit offsets from the tile's first row
  if (x.ld > (int64_t)1 << 25) return fail(FP8_EINVAL, "%s: ld too large (> 2^25 elements)", name);
  if (need_ptr && !x.ptr) return fail(FP8_EINVAL, "%s: null pointer", name);
  if (x.ptr && !aligned16(x.ptr)) return fail(FP8_EALIGN, "%s: pointer not 16-byte aligned", name);
  return FP8_OK;
}
static fp8_status_t check_ptr(const void* p, const char* name) {
  if (!p) return fail(FP8_EINVAL, "%s: null pointer", name);
  if (!aligned16(p)) return fail(FP8_EALIGN, "%s: pointer not 16-byte aligned", name);
  return FP8_OK;
}
static fp8_status_t check_fmt(int f) {
  return (f == FP8_E4M3 || f == FP8_E5M2) ? FP8_OK : fail(FP8_EINVAL, "bad fp8 format");
}

// Bump allocator over a caller buffer (256-byte aligned regions).
struct Carve {
  uint8_t* base;
  size_t off = 0;
  explicit Carve(void* b) : base(static_cast<uint8_t*>(b)) {}
  template <typename T> T* take(size_t bytes) {
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += al(bytes);
    return p;
  }
};

}  // namespace fp8t

using namespace fp8t;

extern "C" {

int fp8_abi_version(void) { return FP8TRAIN_ABI_VERSION; }

fp8_status_t fp8_check_async_error(void) { return check_fault(); }

fp8_status_t fp8_set_knob(const char* name, int value) {
  const int i = knob_index(name);
  if (i < 0) return fail(FP8_EINVAL, "unknown knob '%s'", name ? name : "(null)");
  if (value < kKnobs[i].lo || value > kKnobs[i].hi)
    return fail(FP8_EINVAL, "knob %s: value %d outside [%d, %d]", name, value, kKnobs[i].lo, kKnobs[i].hi);
  g_knobs[i].store(value, std::memory_order_relaxed);
  return FP8_OK;
}
fp8_status_t fp8_get_knob(const char* name, int* value) {
  const int i = knob_index(name);
  if (i < 0) return fail(FP8_EINVAL, "unknown knob '%s'", name ? name : "(null)");
  if (!value) return fail(FP8_EINVAL, "value: null pointer");
  *value = g_knobs[i].load(std::memory_order_relaxed);
  return FP8_OK;
}
void fp8_reset_knobs(void) {
  for (int i = 0; i < KNOB_COUNT; ++i) g_knobs[i].store(kKnobs[i].def, std::memory_order_relaxed);
}
const char* fp8_last_error(void) { return g_err.c_str(); }
uint64_t fp8_launch_count(void) { return g_launches.load(); }

void fp8_profile_enable(int on) { g_prof_on.store(on ? 1 : 0); }

int fp8_profile_collect(int* kinds, float* ms, int max_n) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  int n = 0, rc = 0;
  for (auto& r : g_prof) {
    float t = 0.f;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) rc = -1;
    if (n < max_n) {
      if (kinds) kinds[n] = r.kind;
      if (ms) ms[n] = t;
      ++n;
    }
    g_prof_free.push_back(r.a);
    g_prof_free.push_back(r.b);
  }
  g_prof.clear();
  return rc < 0 ? -1 : n;
}

// ---------------------------------------------------------------------------
// amax
// ---------------------------------------------------------------------------
size_t fp8_amax_workspace_bytes(fp8_hp_t, fp8_gran_t) { return 0; }

fp8_status_t fp8_amax(fp8_hp_t x, fp8_gran_t gran, float* amax_out, void*, size_t, void* stream) {
  FP8T_TRY(check_hp(x, "x"));
  if (!amax_out) return fail(FP8_EINVAL, "amax_out: null pointer");
  int mode;
  size_t n;
  switch (gran) {
    case FP8_GRAN_TENSOR: mode = 1; n = 1; break;
    case FP8_GRAN_ROW: mode = 2; n = x.rows; break;
    case FP8_GRAN_COL: mode = 4; n = x.cols; break;
    default: return fail(FP8_EINVAL, "fp8_amax: gran must be TENSOR, ROW or COL");
  }
  uint32_t* acc = reinterpret_cast<uint32_t*>(amax_out);
  FP8T_CUDA(cudaMemsetAsync(acc, 0, n * 4, S(stream)), "memset amax");
  FP8T_CUDA(launch_amax(x.ptr, x.dtype == FP8_DT_BF16, x.rows, x.cols, x.ld, mode, acc, acc, acc, S(stream)),
            "amax kernel");
  return FP8_OK;
}

fp8_status_t fp8_amax_multi(const fp8_hp_t* xs, int n, float* amax_out, void* stream) {
  if (!xs || !amax_out) return fail(FP8_EINVAL, "xs/amax_out: null pointer");
  if (n < 1 || n > FP8_AMAX_MULTI_MAX) return fail(FP8_EINVAL, "n must be in [1, %d]", FP8_AMAX_MULTI_MAX);
  static_assert(FP8_AMAX_MULTI_MAX == AMAX_MULTI_MAX, "multi-tensor amax capacity");
  AmaxMultiArgs a{};
  a.n = n;
  a.out = reinterpret_cast<uint32_t*>(amax_out);
  a.chunk_start[0] = 0;
  for (int t = 0; t < n; ++t) {
    FP8T_TRY(check_hp(xs[t], "xs[t]"));
    const int64_t es = (int64_t)esize(xs[t].dtype);
    a.ptr[t] = static_cast<const uint8_t*>(xs[t].ptr);
    a.ld_bytes[t] = xs[t].ld * es;
    a.vecs[t] = xs[t].cols * es / 16;
    a.cpr[t] = (a.vecs[t] + 255) / 256;
    a.bf16[t] = xs[t].dtype == FP8_DT_BF16;
    a.chunk_start[t + 1] = a.chunk_start[t] + xs[t].rows * a.cpr[t];
  }
  FP8T_CUDA(cudaMemsetAsync(amax_out, 0, 4 * (size_t)n, S(stream)), "memset amax");
  FP8T_CUDA(launch_amax_multi(a, S(stream)), "amax_multi kernel");
  return FP8_OK;
}

// ---------------------------------------------------------------------------
// cast
// ---------------------------------------------------------------------------
size_t fp8_cast_workspace_bytes(fp8_hp_t x, fp8_gran_t gran) {
  switch (gran) {
    case FP8_GRAN_TENSOR: return al(4);
    case FP8_GRAN_ROW: return al(4 * x.rows);
    case FP8_GRAN_COL: return al(4 * x.cols);
    case FP8_GRAN_ROW_COL: return al(4 * x.rows) + al(4 * x.cols);
    default: return 0;
  }
}

fp8_status_t fp8_cast_scaled(fp8_hp_t x, fp8_mx_round_t mx_round, const float* amax_in, fp8_tensor_t* out,
                             void* ws, size_t ws_bytes, void* stream) {
  FP8T_TRY(check_hp(x, "x"));
  if (!out) return fail(FP8_EINVAL, "out: null pointer");
  FP8T_TRY(check_fmt(out->fmt));
  if (out->rows != x.rows || out->cols != x.cols) return fail(FP8_EINVAL, "out shape != x shape");
  if (!out->q && !out->q_t) return fail(FP8_EINVAL, "out->q and out->q_t are both NULL");
  if (out->q) FP8T_TRY(check_ptr(out->q, "out->q"));
  if (out->q_t) FP8T_TRY(check_ptr(out->q_t, "out->q_t"));
  if (amax_in && out->gran != FP8_GRAN_TENSOR) return fail(FP8_EINVAL, "amax_in is only valid for TENSOR");
  const bool bf16 = x.dtype == FP8_DT_BF16;
  cudaStream_t st = S(stream);
  const int fmt = out->fmt;

  if (out->gran == FP8_GRAN_MX32 || out->gran == FP8_GRAN_MX32_RM) {
    if (x.rows % 128 || x.cols % 128) return fail(FP8_EALIGN, "MX32 needs rows and cols multiples of 128");
    if (mx_round != FP8_MX_FLOOR && mx_round != FP8_MX_RCEIL) return fail(FP8_EINVAL, "bad mx_round");
    if (out->q && !out->scale) return fail(FP8_EINVAL, "MX32: q needs scale");
    if (out->q_t && !out->scale_t) return fail(FP8_EINVAL, "MX32: q_t needs scale_t");
    FP8T_CUDA(launch_mx_cast(x.ptr, bf16, fmt, mx_round == FP8_MX_RCEIL, x.rows, x.cols, x.ld, out->q,
                             static_cast<uint8_t*>(out->scale), out->q_t, static_cast<uint8_t*>(out->scale_t), st,
                             out->gran == FP8_GRAN_MX32),
              "mx cast kernel");
    return FP8_OK;
  }
  if (out->gran < FP8_GRAN_TENSOR || out->gran > FP8_GRAN_ROW_COL) return fail(FP8_EINVAL, "bad gran");
  {
    // amax accumulators come from out->amax / out->amax_t when given, else from ws
    size_t need = 0;
    if (out->gran == FP8_GRAN_ROW_COL) {
      if (!out->amax) need += al(4 * x.rows);
      if (!out->amax_t) need += al(4 * x.cols);
    } else if (!out->amax && !amax_in) {
      need = fp8_cast_workspace_bytes(x, out->gran);
    }
    if (need && (!ws || ws_bytes < need)) return fail(FP8_EWORKSPACE, "workspace too small (%zu < %zu)", ws_bytes, need);
  }
  Carve c(ws);

  if (out->gran == FP8_GRAN_ROW_COL) {
    if (!out->scale || (out->q_t && !out->scale_t)) return fail(FP8_EINVAL, "ROW_COL needs scale (and scale_t)");
    float* ar = out->amax ? out->amax : c.take<float>(4 * x.rows);
    float* ac = out->amax_t ? out->amax_t : c.take<float>(4 * x.cols);
    FP8T_CUDA(cudaMemsetAsync(ar, 0, 4 * x.rows, st), "memset");
    FP8T_CUDA(cudaMemsetAsync(ac, 0, 4 * x.cols, st), "memset");
    FP8T_CUDA(launch_amax(x.ptr, bf16, x.rows, x.cols, x.ld, 6, nullptr, reinterpret_cast<uint32_t*>(ar),
                          reinterpret_cast<uint32_t*>(ac), st),
              "amax kernel");
    FP8T_CUDA(launch_cast(x.ptr, bf16, fmt, x.rows, x.cols, x.ld, out->q ? 2 : 0, out->q_t ? 3 : 0, ar, ac, out->q,
                          out->q_t, static_cast<float*>(out->scale), static_cast<float*>(out->scale_t), st),
              "cast kernel");
    return FP8_OK;
  }

  // TENSOR / ROW / COL: one scale vector shared by q and q_t
  if (!out->scale && !out->scale_t) return fail(FP8_EINVAL, "scale: null pointer");
  const int mode = out->gran == FP8_GRAN_TENSOR ? 1 : (out->gran == FP8_GRAN_ROW ? 2 : 3);
  const int amode = out->gran == FP8_GRAN_TENSOR ? 1 : (out->gran == FP8_GRAN_ROW ? 2 : 4);
  const size_t n = out->gran == FP8_GRAN_TENSOR ? 1 : (out->gran == FP8_GRAN_ROW ? x.rows : x.cols);
  const float* a = amax_in;
  if (!a) {
    float* acc = out->amax ? out->amax : c.take<float>(4 * n);
    FP8T_CUDA(cudaMemsetAsync(acc, 0, 4 * n, st), "memset");
    uint32_t* u = reinterpret_cast<uint32_t*>(acc);
    FP8T_CUDA(launch_amax(x.ptr, bf16, x.rows, x.cols, x.ld, amode, u, u, u, st), "amax kernel");
    a = acc;
  } else if (out->amax && out->amax != amax_in) {
    FP8T_CUDA(cudaMemcpyAsync(out->amax, amax_in, 4, cudaMemcpyDeviceToDevice, st), "copy amax");
  }
  float* sq = static_cast<float*>(out->scale ? out->scale : out->scale_t);
  float* stt = static_cast<float*>(out->scale_t ? out->scale_t : out->scale);
  FP8T_CUDA(launch_cast(x.ptr, bf16, fmt, x.rows, x.cols, x.ld, out->q ? mode : 0, out->q_t ? mode : 0, a, a,
                        out->q, out->q_t, out->q ? sq : nullptr, stt, st),
            "cast kernel");
  return FP8_OK;
}

// ---------------------------------------------------------------------------
// GEMM
// ---------------------------------------------------------------------------
fp8_status_t fp8_gemm(const uint8_t* A, fp8_format_t fmt_a, fp8_major_t major_a, const void* sa, const uint8_t* B,
                      fp8_format_t fmt_b, fp8_major_t major_b, const void* sb, fp8_gran_t gran, int64_t M, int64_t N,
                      int64_t K, int64_t lda, int64_t ldb, void* D, fp8_dtype_t out_dtype, int64_t ldd, void* stream) {
  FP8T_TRY(check_ptr(A, "A"));
  FP8T_TRY(check_ptr(B, "B"));
  FP8T_TRY(check_ptr(D, "D"));
  FP8T_TRY(check_fmt(fmt_a));
  FP8T_TRY(check_fmt(fmt_b));
  if ((major_a != FP8_K_MAJOR && major_a != FP8_MN_MAJOR) || (major_b != FP8_K_MAJOR && major_b != FP8_MN_MAJOR))
    return fail(FP8_EINVAL, "bad operand major");
  if (!sa || !sb) return fail(FP8_EINVAL, "scales: null pointer");
  if (M < 16 || N < 16 || K < 16) return fail(FP8_EINVAL, "M, N, K must be >= 16");
  if (M % 16 || N % 16 || K % 16) return fail(FP8_EALIGN, "M, N, K must be multiples of 16");
  if (M > (1 << 30) || N > (1 << 30) || K > (1 << 30)) return fail(FP8_EINVAL, "dims too large");
  if (lda < (major_a == FP8_K_MAJOR ? K : M) || ldb < (major_b == FP8_K_MAJOR ? K : N) || ldd < N)
    return fail(FP8_EINVAL, "leading dimension too small");
  if (lda % 16 || ldb % 16) return fail(FP8_EALIGN, "lda/ldb must be multiples of 16 bytes");
  if (out_dtype != FP8_DT_BF16 && out_dtype != FP8_DT_F32) return fail(FP8_EINVAL, "bad out_dtype");
  if ((ldd * (int64_t)esize(out_dtype)) % 16) return fail(FP8_EALIGN, "ldd*elem_size must be a multiple of 16");
  int mode;
  if (gran == FP8_GRAN_TENSOR) mode = 0;
  else if (gran == FP8_GRAN_ROW) mode = 1;
  else if (gran == FP8_GRAN_MX32) {
    mode = 2;
    if (M % 128 || N % 128 || K % 128) return fail(FP8_EALIGN, "MX32 GEMM needs M, N, K multiples of 128");
    FP8T_TRY(check_ptr(sa, "sfa"));
    FP8T_TRY(check_ptr(sb, "sfb"));
  } else return fail(FP8_EINVAL, "fp8_gemm: gran must be TENSOR, ROW or MX32");
  GemmProblem p{A, B, (int)fmt_a, (int)fmt_b, major_a == FP8_MN_MAJOR, major_b == FP8_MN_MAJOR,
                sa, sb, mode, M, N, K, lda, ldb, D, out_dtype == FP8_DT_F32, ldd};
  FP8T_CUDA(launch_gemm(p, S(stream)), "gemm kernel");
  return FP8_OK;
}

// ---------------------------------------------------------------------------
// Float8Linear forward / backward
// ---------------------------------------------------------------------------
namespace {

struct Saved {          // written by fwd, read by bwd
  uint8_t* xT;          // tensorwise: Xq [M,K]; rowwise: column-scaled X [M,K] (both row-major, read MN-major
                        // by dW); mxfp8: dim1 copy [K,M] (K-major over M)
  uint8_t* wT;          // tensorwise: Wq [N,K]; rowwise: column-scaled W [N,K] (read MN-major by dX);
                        // mxfp8: dim1 copy [K,N]
  void* sx;             // tensorwise float[1] | rowwise float[K] | mx E8M0 [K x M/32]
  void* sw;             // tensorwise float[1] | rowwise float[K] | mx E8M0 [K x N/32]
};
Saved carve_saved(const fp8_linear_cfg_t* cfg, int64_t M, int64_t N, int64_t K, void* base, size_t* bytes) {
  Carve c(base);
  Saved s;
  s.xT = c.take<uint8_t>((size_t)K * M);
  s.wT = c.take<uint8_t>((size_t)K * N);
  if (cfg->recipe == FP8_RECIPE_TENSORWISE) {
    s.sx = c.take<float>(4);
    s.sw = c.take<float>(4);
  } else if (cfg->recipe == FP8_RECIPE_ROWWISE || cfg->recipe == FP8_RECIPE_ROWWISE_GW_HP) {
    s.sx = c.take<float>(4 * K);
    s.sw = c.take<float>(4 * K);
  } else {
    s.sx = c.take<uint8_t>((size_t)K * M / 32);
    s.sw = c.take<uint8_t>((size_t)K * N / 32);
  }
  if (bytes) *bytes = c.off;
  return s;
}

struct FwdWs {
  uint8_t* xq; uint8_t* wq;
  float* amax;       // tensorwise [2] | rowwise [M + K + N + K]
  float* sxr; float* swr;      // rowwise row scales
  uint8_t* sfx; uint8_t* sfw;  // mx dim0 scales
};
FwdWs carve_fwd(const fp8_linear_cfg_t* cfg, int64_t M, int64_t N, int64_t K, void* base, size_t* bytes) {
  Carve c(base);
  FwdWs w{};
  if (cfg->recipe == FP8_RECIPE_TENSORWISE) {   // codes go straight to the saved buffer
    w.amax = c.take<float>(8);
    if (bytes) *bytes = c.off;
    return w;
  }
  w.xq = c.take<uint8_t>((size_t)M * K);
  w.wq = c.take<uint8_t>((size_t)N * K);
  if (cfg->recipe == FP8_RECIPE_ROWWISE || cfg->recipe == FP8_RECIPE_ROWWISE_GW_HP) {
    w.amax = c.take<float>(4 * (M + K + N + K));
    w.sxr = c.take<float>(4 * M);
    w.swr = c.take<float>(4 * N);
  } else {
    w.sfx = c.take<uint8_t>((size_t)M * K / 32);
    w.sfw = c.take<uint8_t>((size_t)N * K / 32);
  }
  if (bytes) *bytes = c.off;
  return w;
}

struct BwdWs {
  uint8_t* g; uint8_t* gT;   // [M,N], [N,M]
  float* amax;               // tensorwise [1] | rowwise [M + N]
  void* sg; void* sgT;       // tensorwise float[1] | rowwise float[M], float[N] | mx E8M0
};
BwdWs carve_bwd(const fp8_linear_cfg_t* cfg, int64_t M, int64_t N, void* base, size_t* bytes) {
  Carve c(base);
  BwdWs w{};
  w.g = c.take<uint8_t>((size_t)M * N);
  w.gT = cfg->recipe == FP8_RECIPE_TENSORWISE ? nullptr : c.take<uint8_t>((size_t)M * N);
  if (cfg->recipe == FP8_RECIPE_TENSORWISE) {   // dW reads the row-major codes MN-major
    w.amax = c.take<float>(4);
    w.sg = c.take<float>(4);
    w.sgT = w.sg;
  } else if (cfg->recipe == FP8_RECIPE_ROWWISE || cfg->recipe == FP8_RECIPE_ROWWISE_GW_HP) {
    w.amax = c.take<float>(4 * (M + N));
    w.sg = c.take<float>(4 * M);
    w.sgT = c.take<float>(4 * N);
  } else {
    w.sg = c.take<uint8_t>((size_t)M * N / 32);
    w.sgT = c.take<uint8_t>((size_t)M * N / 32);
  }
  if (bytes) *bytes = c.off;
  return w;
}

// Forward-only (inference) workspace: the forward's codes and scales, nothing kept for a backward.
struct InferWs {
  uint8_t* xq; uint8_t* wq;
  void* sx; void* sw;        // tensorwise float[1] | rowwise float[M], float[N] | mx E8M0 dim0
  float* amax;               // tensorwise [2] | rowwise [M + N]
};
InferWs carve_infer(const fp8_linear_cfg_t* cfg, int64_t M, int64_t N, int64_t K, void* base, size_t* bytes) {
  Carve c(base);
  InferWs w{};
  w.xq = c.take<uint8_t>((size_t)M * K);
  w.wq = c.take<uint8_t>((size_t)N * K);
  if (cfg->recipe == FP8_RECIPE_TENSORWISE) {
    w.sx = c.take<float>(4);
    w.sw = c.take<float>(4);
    w.amax = c.take<float>(8);
  } else if (cfg->recipe == FP8_RECIPE_ROWWISE || cfg->recipe == FP8_RECIPE_ROWWISE_GW_HP) {
    w.sx = c.take<float>(4 * M);
    w.sw = c.take<float>(4 * N);
    w.amax = c.take<float>(4 * (M + N));
  } else {
    w.sx = c.take<uint8_t>((size_t)M * K / 32);
    w.sw = c.take<uint8_t>((size_t)N * K / 32);
  }
  if (bytes) *bytes = c.off;
  return w;
}

fp8_status_t check_cfg(const fp8_linear_cfg_t* cfg, int64_t M, int64_t N, int64_t K) {
  if (!cfg) return fail(FP8_EINVAL, "cfg: null pointer");
  if (cfg->recipe < FP8_RECIPE_TENSORWISE || cfg->recipe > FP8_RECIPE_ROWWISE_GW_HP)
    return fail(FP8_EINVAL, "bad recipe");
  FP8T_TRY(check_fmt(cfg->fmt_fwd));
  FP8T_TRY(check_fmt(cfg->fmt_grad));
  if (cfg->out_dtype != FP8_DT_BF16 && cfg->out_dtype != FP8_DT_F32) return fail(FP8_EINVAL, "bad out_dtype");
  if (cfg->mx_round != FP8_MX_FLOOR && cfg->mx_round != FP8_MX_RCEIL) return fail(FP8_EINVAL, "bad mx_round");
  if (M < 16 || N < 16 || K < 16) return fail(FP8_EINVAL, "M, N, K must be >= 16");
  if (M % 16 || N % 16 || K % 16) return fail(FP8_EALIGN, "M, N, K must be multiples of 16");
  if (cfg->recipe == FP8_RECIPE_MXFP8 && (M % 128 || N % 128 || K % 128))
    return fail(FP8_EALIGN, "mxfp8 needs M, N, K multiples of 128");
  return FP8_OK;
}

// Pre-cast weight (FSDP gathers): tensorwise codes + float scale, or MXFP8 dim0 (forward) and
// dim1 (backward dX) codes with E8M0 scales in the layout the backward GEMMs read.
fp8_status_t check_w_fp8(const fp8_linear_cfg_t* cfg, const fp8_tensor_t* w_fp8, int64_t N, int64_t K, bool bwd_dx) {
  if (w_fp8->rows != N || w_fp8->cols != K) return fail(FP8_EINVAL, "w_fp8 shape");
  if (w_fp8->fmt != cfg->fmt_fwd) return fail(FP8_EINVAL, "w_fp8 format != cfg->fmt_fwd");
  if (cfg->recipe == FP8_RECIPE_TENSORWISE) {
    FP8T_TRY(check_ptr(w_fp8->q, "w_fp8->q"));
    if (!w_fp8->scale) return fail(FP8_EINVAL, "w_fp8->scale: null pointer");
    return FP8_OK;
  }
  if (cfg->recipe != FP8_RECIPE_MXFP8) return fail(FP8_EUNSUPPORTED, "w_fp8 needs the tensorwise or mxfp8 recipe");
  if (w_fp8->gran != (mx_transposed() ? FP8_GRAN_MX32 : FP8_GRAN_MX32_RM))
    return fail(FP8_EINVAL, "w_fp8->gran must be FP8_GRAN_MX32_RM (FP8_GRAN_MX32 with knob mx_transposed = 1)");
  if (!bwd_dx) {
    FP8T_TRY(check_ptr(w_fp8->q, "w_fp8->q"));
    if (!w_fp8->scale) return fail(FP8_EINVAL, "w_fp8->scale: null pointer");
  } else {
    FP8T_TRY(check_ptr(w_fp8->q_t, "w_fp8->q_t"));
    if (!w_fp8->scale_t) return fail(FP8_EINVAL, "w_fp8->scale_t: null pointer");
  }
  return FP8_OK;
}

}  // namespace

}  // extern "C"

// Training forward of one linear (fp8_linear_fwd_ex with `saved`, and each member of
// fp8_linear_fwd_shared).  X's operands go to / come from `svx` (its backward copy) and `fw` (its
// forward copy, row scales / E8M0), W's to `svw` and `fw`.  cast_x = false: X's amax and casts were
// already written by the previous member of a shared-input group (same x, same fw / svx), so only
// W is cast here -- the bytes are the ones a separate fp8_linear_fwd would write.  W's forward
// operand goes to fw.wq / fw.swr / fw.sfw (a group passes each member its own slice) and its amax to
// the fw.amax slots after X's (reused member after member: each W amax is consumed by W's cast).
static fp8_status_t linear_fwd_train(const fp8_linear_cfg_t* cfg, fp8_hp_t x, const float* x_amax, fp8_hp_t w,
                                     const fp8_tensor_t* w_fp8, void* y, float* y_amax, const Saved& svx,
                                     const Saved& svw, const FwdWs& fw, bool cast_x, cudaStream_t st,
                                     GemmProblem* defer = nullptr, bool cast_done = false) {
  const int64_t M = x.rows, K = x.cols, N = w.rows;
  const bool xb = x.dtype == FP8_DT_BF16, wb = w.dtype == FP8_DT_BF16;
  const int ff = cfg->fmt_fwd;
  const int of32 = cfg->out_dtype == FP8_DT_F32;
  uint32_t* yam = reinterpret_cast<uint32_t*>(y_amax);
  // defer: hand the GEMM back to the caller (a shared-input group launches its members' GEMMs together)
  auto fwd_gemm = [&](const GemmProblem& p) -> fp8_status_t {
    if (defer) {
      *defer = p;
      return FP8_OK;
    }
    if (yam) FP8T_CUDA(cudaMemsetAsync(yam, 0, 4, st), "memset y_amax");
    FP8T_CUDA(launch_gemm(p, st), "gemm fwd");
    return FP8_OK;
  };
  if (cfg->recipe == FP8_RECIPE_TENSORWISE) {
    // row-major codes only: the backward GEMMs read them MN-major (no transposed copies)
    uint32_t* ax = reinterpret_cast<uint32_t*>(fw.amax);
    uint32_t* aw = ax + 1;
    const float* axp = x_amax ? x_amax : fw.amax;
    const uint8_t* wq = svw.wT;
    FP8T_CUDA(cudaMemsetAsync(cast_x ? ax : aw, 0, cast_x ? 8 : 4, st), "memset");
    // amax X and W by one launch, then X and W cast by one launch (measured on c2: casts 0.165 ->
    // 0.158 ms per step); knob tw_dual = 0 keeps four launches (X's cast right after its amax).
    // x_amax: amax(X) precomputed by X's producer (e.g. the previous layer's epilogue) -> no amax pass
    const bool tw_dual = knob(KNOB_TW_DUAL) == 1;
    if (!cast_x) {
      if (w_fp8) {
        wq = w_fp8->q;
        FP8T_CUDA(cudaMemcpyAsync(svw.sw, w_fp8->scale, 4, cudaMemcpyDeviceToDevice, st), "copy w scale");
      } else {
        FP8T_CUDA(launch_amax(w.ptr, wb, N, K, w.ld, 1, aw, nullptr, nullptr, st), "amax w");
        FP8T_CUDA(launch_cast(w.ptr, wb, ff, N, K, w.ld, 1, 0, fw.amax + 1, fw.amax + 1, svw.wT, nullptr,
                              (float*)svw.sw, nullptr, st),
                  "cast w");
      }
    } else if (tw_dual && !w_fp8 && xb == wb) {
      cudaError_t e = cudaErrorNotSupported;
      if (!x_amax && x.ld == K && w.ld == K)
        e = launch_amax_flat_dual(x.ptr, M * K, ax, w.ptr, N * K, aw, xb, st);
      if (e != cudaErrorNotSupported) {
        FP8T_CUDA(e, "amax x, w");
      } else {
        if (!x_amax) FP8T_CUDA(launch_amax(x.ptr, xb, M, K, x.ld, 1, ax, nullptr, nullptr, st), "amax x");
        FP8T_CUDA(launch_amax(w.ptr, wb, N, K, w.ld, 1, aw, nullptr, nullptr, st), "amax w");
      }
      CastDual cd{};
      cd.x[0] = x.ptr; cd.R[0] = M; cd.C[0] = K; cd.ld[0] = x.ld; cd.amax_q[0] = axp; cd.amax_t[0] = axp;
      cd.q[0] = svx.xT; cd.scale_q[0] = (float*)svx.sx;
      cd.x[1] = w.ptr; cd.R[1] = N; cd.C[1] = K; cd.ld[1] = w.ld; cd.amax_q[1] = fw.amax + 1;
      cd.amax_t[1] = fw.amax + 1; cd.q[1] = svw.wT; cd.scale_q[1] = (float*)svw.sw;
      FP8T_CUDA(launch_cast_dual(cd, xb, ff, 1, 0, st), "cast x, w");
    } else {
      if (!x_amax) FP8T_CUDA(launch_amax(x.ptr, xb, M, K, x.ld, 1, ax, nullptr, nullptr, st), "amax x");
      FP8T_CUDA(launch_cast(x.ptr, xb, ff, M, K, x.ld, 1, 0, axp, axp, svx.xT, nullptr, (float*)svx.sx, nullptr, st),
                "cast x");
      if (w_fp8) {
        wq = w_fp8->q;
        FP8T_CUDA(cudaMemcpyAsync(svw.sw, w_fp8->scale, 4, cudaMemcpyDeviceToDevice, st), "copy w scale");
      } else {
        FP8T_CUDA(launch_amax(w.ptr, wb, N, K, w.ld, 1, aw, nullptr, nullptr, st), "amax w");
        FP8T_CUDA(launch_cast(w.ptr, wb, ff, N, K, w.ld, 1, 0, fw.amax + 1, fw.amax + 1, svw.wT, nullptr,
                              (float*)svw.sw, nullptr, st),
                  "cast w");
      }
    }
    GemmProblem p{svx.xT, wq, ff, ff, 0, 0, svx.sx, svw.sw, 0, M, N, K, K, K, y, of32, N, 0, yam};
    FP8T_TRY(fwd_gemm(p));
  } else if (cfg->recipe == FP8_RECIPE_ROWWISE || cfg->recipe == FP8_RECIPE_ROWWISE_GW_HP) {
    const bool gw_hp = cfg->recipe == FP8_RECIPE_ROWWISE_GW_HP;   // X's column-scaled copy unused
    float* axr = fw.amax;
    float* axc = axr + M;
    float* awr = axc + K;
    float* awc = awr + N;
    if (cast_done) {   // a shared-input group cast X and every W_i by one amax and one cast launch
      GemmProblem p{fw.xq, fw.wq, ff, ff, 0, 0, fw.sxr, fw.swr, 1, M, N, K, K, K, y, of32, N, 0, yam};
      return fwd_gemm(p);
    }
    if (!cast_x) {   // X's row / column amax, codes and scales are already in fw / svx
      FP8T_CUDA(cudaMemsetAsync(awr, 0, 4 * (N + K), st), "memset");
      FP8T_CUDA(launch_amax(w.ptr, wb, N, K, w.ld, 6, nullptr, (uint32_t*)awr, (uint32_t*)awc, st), "amax w");
      FP8T_CUDA(launch_cast(w.ptr, wb, ff, N, K, w.ld, 2, 5, awr, awc, fw.wq, svw.wT, fw.swr, (float*)svw.sw, st),
                "cast w");
      GemmProblem p{fw.xq, fw.wq, ff, ff, 0, 0, fw.sxr, fw.swr, 1, M, N, K, K, K, y, of32, N, 0, yam};
      return fwd_gemm(p);
    }
    FP8T_CUDA(cudaMemsetAsync(fw.amax, 0, 4 * (M + K + N + K), st), "memset");
    // X and W in one amax launch and one cast launch where the shapes allow (the small weights of
    // e.g. the wk/wv projections then cost no launch ramp and tail of their own); rowwise_gw_hp
    // needs different scale modes for X and W, so it keeps separate launches
    bool dual = false;
    if (!gw_hp && xb && wb) {
      const cudaError_t e = launch_amax_dual(x.ptr, M, K, x.ld, w.ptr, N, K, w.ld, 6, (uint32_t*)axr, (uint32_t*)axc,
                                             (uint32_t*)awr, (uint32_t*)awc, st);
      if (e != cudaErrorNotSupported) FP8T_CUDA(e, "amax x, w");
      dual = e == cudaSuccess;
    }
    if (!dual) {
      FP8T_CUDA(launch_amax(x.ptr, xb, M, K, x.ld, gw_hp ? 2 : 6, nullptr, (uint32_t*)axr, (uint32_t*)axc, st),
                "amax x");
      FP8T_CUDA(launch_amax(w.ptr, wb, N, K, w.ld, 6, nullptr, (uint32_t*)awr, (uint32_t*)awc, st), "amax w");
    }
    // row-scaled codes for the forward GEMM; column-scaled codes written row-major for the
    // backward GEMMs (read MN-major, no transposed copy)
    if (!gw_hp && xb == wb) {
      CastDual cd{};
      cd.x[0] = x.ptr; cd.R[0] = M; cd.C[0] = K; cd.ld[0] = x.ld; cd.amax_q[0] = axr; cd.amax_t[0] = axc;
      cd.q[0] = fw.xq; cd.qt[0] = svx.xT; cd.scale_q[0] = fw.sxr; cd.scale_t[0] = (float*)svx.sx;
      cd.x[1] = w.ptr; cd.R[1] = N; cd.C[1] = K; cd.ld[1] = w.ld; cd.amax_q[1] = awr; cd.amax_t[1] = awc;
      cd.q[1] = fw.wq; cd.qt[1] = svw.wT; cd.scale_q[1] = fw.swr; cd.scale_t[1] = (float*)svw.sw;
      FP8T_CUDA(launch_cast_dual(cd, xb, ff, 2, 5, st), "cast x, w");
    } else {
      FP8T_CUDA(launch_cast(x.ptr, xb, ff, M, K, x.ld, 2, gw_hp ? 0 : 5, axr, axc, fw.xq, gw_hp ? nullptr : svx.xT,
                            fw.sxr, gw_hp ? nullptr : (float*)svx.sx, st),
                "cast x");
      FP8T_CUDA(launch_cast(w.ptr, wb, ff, N, K, w.ld, 2, 5, awr, awc, fw.wq, svw.wT, fw.swr, (float*)svw.sw, st),
                "cast w");
    }
    GemmProblem p{fw.xq, fw.wq, ff, ff, 0, 0, fw.sxr, fw.swr, 1, M, N, K, K, K, y, of32, N, 0, yam};
    FP8T_TRY(fwd_gemm(p));
  } else {
    const bool rc = cfg->mx_round == FP8_MX_RCEIL, tr = mx_transposed();
    if (cast_x)
      FP8T_CUDA(launch_mx_cast(x.ptr, xb, ff, rc, M, K, x.ld, fw.xq, fw.sfx, svx.xT, (uint8_t*)svx.sx, st, tr),
                "mx cast x");
    // pre-gathered weight (fp8_fsdp_allgather_mx): its dim0 copy feeds this GEMM and its dim1 copy
    // the backward, so nothing of W is cast or saved here
    if (!w_fp8)
      FP8T_CUDA(launch_mx_cast(w.ptr, wb, ff, rc, N, K, w.ld, fw.wq, fw.sfw, svw.wT, (uint8_t*)svw.sw, st, tr),
                "mx cast w");
    const uint8_t* wq = w_fp8 ? w_fp8->q : fw.wq;
    const void* swp = w_fp8 ? w_fp8->scale : fw.sfw;
    GemmProblem p{fw.xq, wq, ff, ff, 0, 0, fw.sfx, swp, 2, M, N, K, K, K, y, of32, N, 0, yam};
    FP8T_TRY(fwd_gemm(p));
  }
  return FP8_OK;
}


extern "C" {

size_t fp8_linear_saved_bytes(const fp8_linear_cfg_t* cfg, int64_t M, int64_t N, int64_t K) {
  if (!cfg) return 0;
  size_t b = 0;
  carve_saved(cfg, M, N, K, nullptr, &b);
  return b;
}

fp8_status_t fp8_linear_buffers(const fp8_linear_cfg_t* cfg, int64_t M, int64_t N, int64_t K, void* saved,
                                void* ws, fp8_linear_buffers_t* out) {
  if (!out) return fail(FP8_EINVAL, "out: null pointer");
  FP8T_TRY(check_cfg(cfg, M, N, K));
  FP8T_TRY(check_ptr(saved, "saved"));
  FP8T_TRY(check_ptr(ws, "ws"));
  *out = fp8_linear_buffers_t{};
  const Saved sv = carve_saved(cfg, M, N, K, saved, nullptr);
  const FwdWs fw = carve_fwd(cfg, M, N, K, ws, nullptr);
  const BwdWs bw = carve_bwd(cfg, M, N, ws, nullptr);
  out->x_bwd = sv.xT; out->x_bwd_scale = sv.sx;
  out->w_bwd = sv.wT; out->w_bwd_scale = sv.sw;
  out->dy_dx = bw.g; out->dy_dx_scale = bw.sg;
  out->dy_dw = bw.gT; out->dy_dw_scale = bw.sgT;
  out->amax_fwd = fw.amax; out->amax_bwd = bw.amax;
  if (cfg->recipe == FP8_RECIPE_TENSORWISE) {
    out->x_fwd = sv.xT; out->x_fwd_scale = sv.sx;
    out->w_fwd = sv.wT; out->w_fwd_scale = sv.sw;
    out->dy_dw = bw.g; out->dy_dw_scale = bw.sg;
  } else if (cfg->recipe == FP8_RECIPE_MXFP8) {
    out->x_fwd = fw.xq; out->x_fwd_scale = fw.sfx;
    out->w_fwd = fw.wq; out->w_fwd_scale = fw.sfw;
    out->amax_fwd = out->amax_bwd = nullptr;
    out->bwd_transposed = mx_transposed() ? 1 : 0;
  } else {
    out->x_fwd = fw.xq; out->x_fwd_scale = fw.sxr;
    out->w_fwd = fw.wq; out->w_fwd_scale = fw.swr;
    if (cfg->recipe == FP8_RECIPE_ROWWISE_GW_HP) {
      out->x_bwd = nullptr; out->x_bwd_scale = nullptr;
      out->dy_dw = nullptr; out->dy_dw_scale = nullptr;
    }
  }
  return FP8_OK;
}

size_t fp8_linear_infer_workspace_bytes(const fp8_linear_cfg_t* cfg, int64_t M, int64_t N, int64_t K) {
  if (!cfg) return 0;
  size_t b = 0;
  carve_infer(cfg, M, N, K, nullptr, &b);
  return b;
}

size_t fp8_linear_workspace_bytes(const fp8_linear_cfg_t* cfg, int64_t M, int64_t N, int64_t K) {
  if (!cfg) return 0;
  size_t f = 0, b = 0;
  carve_fwd(cfg, M, N, K, nullptr, &f);
  carve_bwd(cfg, M, N, nullptr, &b);
  return f > b ? f : b;
}

fp8_status_t fp8_linear_fwd(const fp8_linear_cfg_t* cfg, fp8_hp_t x, fp8_hp_t w, const fp8_tensor_t* w_fp8,
                            void* y, void* saved, void* ws, size_t ws_bytes, void* stream) {
  return fp8_linear_fwd_ex(cfg, x, nullptr, w, w_fp8, y, nullptr, saved, ws, ws_bytes, stream);
}

fp8_status_t fp8_linear_fwd_ex(const fp8_linear_cfg_t* cfg, fp8_hp_t x, const float* x_amax, fp8_hp_t w,
                               const fp8_tensor_t* w_fp8, void* y, float* y_amax, void* saved, void* ws,
                               size_t ws_bytes, void* stream) {
  FP8T_TRY(check_hp(x, "x"));
  FP8T_TRY(check_hp(w, "w", w_fp8 == nullptr));
  const int64_t M = x.rows, K = x.cols, N = w.rows;
  if (w.cols != K) return fail(FP8_EINVAL, "w.cols != x.cols");
  FP8T_TRY(check_cfg(cfg, M, N, K));
  FP8T_TRY(check_ptr(y, "y"));
  if (saved) FP8T_TRY(check_ptr(saved, "saved"));
  FP8T_TRY(check_ptr(ws, "ws"));
  const size_t need = saved ? fp8_linear_workspace_bytes(cfg, M, N, K) : fp8_linear_infer_workspace_bytes(cfg, M, N, K);
  if (ws_bytes < need) return fail(FP8_EWORKSPACE, "workspace too small (%zu < %zu)", ws_bytes, need);
  if (w_fp8) FP8T_TRY(check_w_fp8(cfg, w_fp8, N, K, false));
  if (x_amax && cfg->recipe != FP8_RECIPE_TENSORWISE)
    return fail(FP8_EUNSUPPORTED, "x_amax (precomputed tensor amax) needs the tensorwise recipe");
  cudaStream_t st = S(stream);
  const bool xb = x.dtype == FP8_DT_BF16, wb = w.dtype == FP8_DT_BF16;
  const int ff = cfg->fmt_fwd;
  const int of32 = cfg->out_dtype == FP8_DT_F32;
  uint32_t* yam = reinterpret_cast<uint32_t*>(y_amax);
  // y_amax is zeroed right before the forward GEMM, after every cast has read x_amax, so a caller
  // chaining layers through one buffer (x_amax == y_amax) gets X cast with the incoming amax
  auto fwd_gemm = [&](const GemmProblem& p) -> fp8_status_t {
    if (yam) FP8T_CUDA(cudaMemsetAsync(yam, 0, 4, st), "memset y_amax");
    FP8T_CUDA(launch_gemm(p, st), "gemm fwd");
    return FP8_OK;
  };

  if (!saved) {
    // forward-only FP8 (inference / float8 dynamic activation + weight, PAPER.md:470-471, 636:
    // "same configurations as FP8 training"): only the forward operands are cast
    InferWs iw = carve_infer(cfg, M, N, K, ws, nullptr);
    if (cfg->recipe == FP8_RECIPE_TENSORWISE) {
      uint32_t* ax = reinterpret_cast<uint32_t*>(iw.amax);
      FP8T_CUDA(cudaMemsetAsync(ax, 0, 8, st), "memset");
      if (!x_amax) FP8T_CUDA(launch_amax(x.ptr, xb, M, K, x.ld, 1, ax, nullptr, nullptr, st), "amax x");
      const float* axp = x_amax ? x_amax : iw.amax;
      FP8T_CUDA(launch_cast(x.ptr, xb, ff, M, K, x.ld, 1, 0, axp, axp, iw.xq, nullptr, (float*)iw.sx, nullptr, st),
                "cast x");
      const uint8_t* wq = iw.wq;
      const void* swp = iw.sw;
      if (w_fp8) {
        wq = w_fp8->q;
        swp = w_fp8->scale;
      } else {
        FP8T_CUDA(launch_amax(w.ptr, wb, N, K, w.ld, 1, ax + 1, nullptr, nullptr, st), "amax w");
        FP8T_CUDA(launch_cast(w.ptr, wb, ff, N, K, w.ld, 1, 0, iw.amax + 1, iw.amax + 1, iw.wq, nullptr,
                              (float*)iw.sw, nullptr, st),
                  "cast w");
      }
      GemmProblem p{iw.xq, wq, ff, ff, 0, 0, iw.sx, swp, 0, M, N, K, K, K, y, of32, N, 0, yam};
      FP8T_TRY(fwd_gemm(p));
    } else if (cfg->recipe == FP8_RECIPE_ROWWISE || cfg->recipe == FP8_RECIPE_ROWWISE_GW_HP) {   // PerRow
      float* axr = iw.amax;
      float* awr = axr + M;
      FP8T_CUDA(cudaMemsetAsync(iw.amax, 0, 4 * (M + N), st), "memset");
      FP8T_CUDA(launch_amax(x.ptr, xb, M, K, x.ld, 2, nullptr, (uint32_t*)axr, nullptr, st), "amax x");
      FP8T_CUDA(launch_amax(w.ptr, wb, N, K, w.ld, 2, nullptr, (uint32_t*)awr, nullptr, st), "amax w");
      FP8T_CUDA(launch_cast(x.ptr, xb, ff, M, K, x.ld, 2, 0, axr, axr, iw.xq, nullptr, (float*)iw.sx, nullptr, st),
                "cast x");
      FP8T_CUDA(launch_cast(w.ptr, wb, ff, N, K, w.ld, 2, 0, awr, awr, iw.wq, nullptr, (float*)iw.sw, nullptr, st),
                "cast w");
      GemmProblem p{iw.xq, iw.wq, ff, ff, 0, 0, iw.sx, iw.sw, 1, M, N, K, K, K, y, of32, N, 0, yam};
      FP8T_TRY(fwd_gemm(p));
    } else {   // MXFP8: dim0 only
      const bool rc = cfg->mx_round == FP8_MX_RCEIL;
      FP8T_CUDA(launch_mx_cast(x.ptr, xb, ff, rc, M, K, x.ld, iw.xq, (uint8_t*)iw.sx, nullptr, nullptr, st), "mx x");
      if (!w_fp8)
        FP8T_CUDA(launch_mx_cast(w.ptr, wb, ff, rc, N, K, w.ld, iw.wq, (uint8_t*)iw.sw, nullptr, nullptr, st), "mx w");
      const uint8_t* wq = w_fp8 ? w_fp8->q : iw.wq;
      const void* swp = w_fp8 ? w_fp8->scale : iw.sw;
      GemmProblem p{iw.xq, wq, ff, ff, 0, 0, iw.sx, swp, 2, M, N, K, K, K, y, of32, N, 0, yam};
      FP8T_TRY(fwd_gemm(p));
    }
    return FP8_OK;
  }

  const Saved sv = carve_saved(cfg, M, N, K, saved, nullptr);
  const FwdWs fw = carve_fwd(cfg, M, N, K, ws, nullptr);
  return linear_fwd_train(cfg, x, x_amax, w, w_fp8, y, y_amax, sv, sv, fw, true, st);
}

fp8_status_t fp8_linear_bwd(const fp8_linear_cfg_t* cfg, fp8_hp_t dy, fp8_hp_t x, const void* saved,
                            const fp8_tensor_t* w_fp8, void* dx, void* dw, void* ws, size_t ws_bytes, void* stream) {
  return fp8_linear_bwd_ex(cfg, dy, nullptr, x, saved, w_fp8, dx, nullptr, dw, ws, ws_bytes, stream);
}

static fp8_status_t linear_bwd_impl(const fp8_linear_cfg_t* cfg, fp8_hp_t dy, const float* dy_amax, fp8_hp_t x,
                                    const void* saved, const fp8_tensor_t* w_fp8, void* dx, float* dx_amax, void* dw,
                                    void* ws, size_t ws_bytes, void* stream, fp8_p2p_t rs_win, int rs_nranks,
                                    const void* saved_x = nullptr, int64_t n_x = 0, const BwdWs* bw_in = nullptr,
                                    std::vector<GemmProblem>* defer = nullptr, bool cast_done = false);

// Linears sharing one input (see fp8train.h): X is cast once by member 0, members 1..n-1 cast W only;
// every member's GEMMs run in one persistent launch (up to GEMM_MAX_PROBS problems per launch).
namespace {

struct SharedDims {
  int64_t M = 0, K = 0, nsum = 0, nmax = 0;
  int64_t pre[FP8_SHARED_MAX + 1] = {};   // prefix sums of N_i
};

// Group backward workspace: every member's dY operands side by side (they must all be resident when the
// group's GEMMs run); the amax scratch is reused member after member (each dY amax feeds its own cast).
struct BwdGroupWs {
  uint8_t* g; uint8_t* gT;   // [M, nsum] each, member i at column block pre[i] (as M x N_i arrays)
  float* amax;               // tensorwise [1] | rowwise [M + nmax]
  void* sg; void* sgT;       // tensorwise float[n] | rowwise float[n * M], float[nsum] | mx E8M0 [M * nsum / 32] x 2
};
BwdGroupWs carve_bwd_group(const fp8_linear_cfg_t* cfg, const SharedDims& d, int n, void* base, size_t* bytes) {
  Carve c(base);
  BwdGroupWs w{};
  const int64_t M = d.M, S = d.nsum;
  w.g = c.take<uint8_t>((size_t)M * S);
  w.gT = cfg->recipe == FP8_RECIPE_TENSORWISE ? nullptr : c.take<uint8_t>((size_t)M * S);
  if (cfg->recipe == FP8_RECIPE_TENSORWISE) {
    w.amax = c.take<float>(4);
    w.sg = c.take<float>(4 * n);
    w.sgT = w.sg;
  } else if (cfg->recipe == FP8_RECIPE_ROWWISE || cfg->recipe == FP8_RECIPE_ROWWISE_GW_HP) {
    w.amax = c.take<float>(4 * (M + d.nmax));
    w.sg = c.take<float>(4 * (size_t)n * M);
    w.sgT = c.take<float>(4 * S);
  } else {
    w.sg = c.take<uint8_t>((size_t)M * S / 32);
    w.sgT = c.take<uint8_t>((size_t)M * S / 32);
  }
  if (bytes) *bytes = c.off;
  return w;
}
BwdWs bwd_member(const fp8_linear_cfg_t* cfg, const BwdGroupWs& w, const SharedDims& d, int i) {
  const int64_t M = d.M, off = d.pre[i];
  BwdWs b{};
  b.g = w.g + M * off;
  b.gT = w.gT ? w.gT + M * off : nullptr;
  b.amax = w.amax;
  if (cfg->recipe == FP8_RECIPE_TENSORWISE) {
    b.sg = b.sgT = static_cast<float*>(w.sg) + i;
  } else if (cfg->recipe == FP8_RECIPE_ROWWISE || cfg->recipe == FP8_RECIPE_ROWWISE_GW_HP) {
    b.sg = static_cast<float*>(w.sg) + (size_t)i * M;
    b.sgT = static_cast<float*>(w.sgT) + off;
  } else {
    b.sg = static_cast<uint8_t*>(w.sg) + M * off / 32;
    b.sgT = static_cast<uint8_t*>(w.sgT) + M * off / 32;
  }
  return b;
}
// Group forward workspace = carve_fwd for N = nsum: X's operands once, W_i's forward operands at row pre[i].
FwdWs fwd_member(const fp8_linear_cfg_t* cfg, const FwdWs& f, const SharedDims& d, int i) {
  FwdWs m = f;
  const int64_t off = d.pre[i];
  if (cfg->recipe == FP8_RECIPE_TENSORWISE) return m;   // W's codes and scale live in its saved buffer
  m.wq = f.wq + off * d.K;
  if (cfg->recipe == FP8_RECIPE_MXFP8) m.sfw = f.sfw + off * d.K / 32;
  else m.swr = f.swr + off;
  return m;
}
// Batched group casts (rowwise; knob group_batch): X and every W_i (forward), every member's dY (backward)
// go through ONE amax launch and ONE cast launch, so each tensor needs its own row / column amax slots
// while the launch runs: forward [M + K] for X then [N_i + K] per W_i, backward [M + N_i] per dY_i,
// placed after the forward / backward workspace regions.
bool group_batchable(const fp8_linear_cfg_t* cfg, int n) {
  return cfg->recipe == FP8_RECIPE_ROWWISE && n + 1 <= AMAX_RC_MAX && n + 1 <= CAST_MULTI_MAX;
}
size_t group_fwd_amax_floats(const fp8_linear_cfg_t* cfg, const SharedDims& d, int n) {
  return group_batchable(cfg, n) ? (size_t)(d.M + d.K + d.nsum + (int64_t)n * d.K) : 0;
}
size_t group_bwd_amax_floats(const fp8_linear_cfg_t* cfg, const SharedDims& d, int n) {
  return group_batchable(cfg, n) ? (size_t)((int64_t)n * d.M + d.nsum) : 0;
}
size_t shared_ws_bytes(const fp8_linear_cfg_t* cfg, const SharedDims& d, int n) {
  size_t f = 0, b = 0;
  carve_fwd(cfg, d.M, d.nsum, d.K, nullptr, &f);
  carve_bwd_group(cfg, d, n, nullptr, &b);
  f += al(4 * group_fwd_amax_floats(cfg, d, n));
  b += al(4 * group_bwd_amax_floats(cfg, d, n));
  return f > b ? f : b;
}
float* group_fwd_amax(const fp8_linear_cfg_t* cfg, const SharedDims& d, void* ws) {
  size_t f = 0;
  carve_fwd(cfg, d.M, d.nsum, d.K, nullptr, &f);
  return reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + f);
}
float* group_bwd_amax(const fp8_linear_cfg_t* cfg, const SharedDims& d, int n, void* ws) {
  size_t b = 0;
  carve_bwd_group(cfg, d, n, nullptr, &b);
  return reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + b);
}
// Launch a group's GEMM problems: FP8 and BF16 (rowwise_gw_hp dW) kinds apart, GEMM_MAX_PROBS per launch.
fp8_status_t launch_group(const std::vector<GemmProblem>& ps, cudaStream_t st) {
  for (int bf = 0; bf < 2; ++bf) {
    std::vector<GemmProblem> q;
    for (const GemmProblem& p : ps)
      if (p.bf16_in == bf) q.push_back(p);
    for (size_t i = 0; i < q.size(); i += GEMM_MAX_PROBS) {
      const int n = (int)std::min(q.size() - i, (size_t)GEMM_MAX_PROBS);
      FP8T_CUDA(launch_gemms(q.data() + i, n, st), "shared-input group gemms");
    }
  }
  return FP8_OK;
}

}  // namespace

size_t fp8_linear_shared_workspace_bytes(const fp8_linear_cfg_t* cfg, int64_t M, int64_t K, int n, const int64_t* N) {
  if (!cfg || !N || n < 1 || n > FP8_SHARED_MAX) return 0;
  SharedDims d;
  d.M = M;
  d.K = K;
  for (int i = 0; i < n; ++i) {
    d.pre[i + 1] = d.pre[i] + N[i];
    d.nmax = N[i] > d.nmax ? N[i] : d.nmax;
  }
  d.nsum = d.pre[n];
  return shared_ws_bytes(cfg, d, n);
}

fp8_status_t fp8_linear_fwd_shared(const fp8_linear_cfg_t* cfg, fp8_hp_t x, int n, const fp8_hp_t* w, void* const* y,
                                   void* const* saved, void* ws, size_t ws_bytes, void* stream) {
  FP8T_TRY(check_hp(x, "x"));
  if (n < 1 || n > FP8_SHARED_MAX) return fail(FP8_EINVAL, "n must be in [1, %d]", FP8_SHARED_MAX);
  if (!w || !y || !saved) return fail(FP8_EINVAL, "w / y / saved: null array");
  SharedDims d;
  d.M = x.rows;
  d.K = x.cols;
  for (int i = 0; i < n; ++i) {   // every argument is checked before the first launch
    FP8T_TRY(check_hp(w[i], "w[i]"));
    if (w[i].cols != d.K) return fail(FP8_EINVAL, "w[%d].cols != x.cols", i);
    FP8T_TRY(check_cfg(cfg, d.M, w[i].rows, d.K));
    FP8T_TRY(check_ptr(y[i], "y[i]"));
    FP8T_TRY(check_ptr(saved[i], "saved[i]"));
    d.pre[i + 1] = d.pre[i] + w[i].rows;
    d.nmax = w[i].rows > d.nmax ? w[i].rows : d.nmax;
  }
  d.nsum = d.pre[n];
  FP8T_TRY(check_ptr(ws, "ws"));
  const size_t need = shared_ws_bytes(cfg, d, n);
  if (ws_bytes < need) return fail(FP8_EWORKSPACE, "workspace too small (%zu < %zu)", ws_bytes, need);
  cudaStream_t st = S(stream);
  // X's forward codes and row scales / E8M0 stay where member 0 wrote them; W_i's go to its slice
  const FwdWs fw = carve_fwd(cfg, d.M, d.nsum, d.K, ws, nullptr);
  const Saved sv0 = carve_saved(cfg, d.M, w[0].rows, d.K, saved[0], nullptr);
  // rowwise: X's and every W_i's row / column amax by one launch, their row-scaled forward codes and
  // column-scaled backward copies by one cast launch (the bytes separate linears write)
  bool batched = false;
  bool all_bf16 = x.dtype == FP8_DT_BF16;
  for (int i = 0; i < n; ++i) all_bf16 = all_bf16 && w[i].dtype == FP8_DT_BF16;
  if (group_batchable(cfg, n) && all_bf16 && knob(KNOB_GROUP_BATCH) == 1) {
    float* am = group_fwd_amax(cfg, d, ws);
    FP8T_CUDA(cudaMemsetAsync(am, 0, 4 * group_fwd_amax_floats(cfg, d, n), st), "memset group amax");
    AmaxRCTensor ts[AMAX_RC_MAX];
    CastMulti cm{};
    cm.n = n + 1;
    float* p = am;
    for (int k = 0; k <= n; ++k) {
      const fp8_hp_t& t = k ? w[k - 1] : x;
      float* ar = p;
      float* ac = p + t.rows;
      p = ac + d.K;
      ts[k] = AmaxRCTensor{t.ptr, t.rows, t.cols, t.ld, reinterpret_cast<uint32_t*>(ar), reinterpret_cast<uint32_t*>(ac)};
      cm.x[k] = t.ptr; cm.R[k] = t.rows; cm.C[k] = t.cols; cm.ld[k] = t.ld;
      cm.amax_q[k] = ar; cm.amax_t[k] = ac;
      if (k == 0) {
        cm.q[k] = fw.xq; cm.qt[k] = sv0.xT; cm.scale_q[k] = fw.sxr; cm.scale_t[k] = static_cast<float*>(sv0.sx);
      } else {
        const FwdWs fm = fwd_member(cfg, fw, d, k - 1);
        const Saved svk = carve_saved(cfg, d.M, t.rows, d.K, saved[k - 1], nullptr);
        cm.q[k] = fm.wq; cm.qt[k] = svk.wT; cm.scale_q[k] = fm.swr; cm.scale_t[k] = static_cast<float*>(svk.sw);
      }
    }
    const cudaError_t e = launch_amax_rc(ts, n + 1, 6, st);
    if (e != cudaErrorNotSupported) {
      FP8T_CUDA(e, "group amax");
      FP8T_CUDA(launch_cast_dual(cm, true, cfg->fmt_fwd, 2, 5, st), "group cast");
      batched = true;
    }
  }
  std::vector<GemmProblem> ps(n);
  for (int i = 0; i < n; ++i) {
    const Saved svi = i ? carve_saved(cfg, d.M, w[i].rows, d.K, saved[i], nullptr) : sv0;
    FP8T_TRY(linear_fwd_train(cfg, x, nullptr, w[i], nullptr, y[i], nullptr, sv0, svi, fwd_member(cfg, fw, d, i),
                              i == 0, st, &ps[i], batched));
  }
  return launch_group(ps, st);
}

fp8_status_t fp8_linear_bwd_shared(const fp8_linear_cfg_t* cfg, int n, const fp8_hp_t* dy, fp8_hp_t x,
                                   const void* const* saved, void* const* dx, void* const* dw, void* ws,
                                   size_t ws_bytes, void* stream) {
  if (n < 1 || n > FP8_SHARED_MAX) return fail(FP8_EINVAL, "n must be in [1, %d]", FP8_SHARED_MAX);
  if (!dy || !saved) return fail(FP8_EINVAL, "dy / saved: null array");
  const bool gw_hp = cfg && cfg->recipe == FP8_RECIPE_ROWWISE_GW_HP;
  SharedDims d;
  d.M = x.rows;
  d.K = x.cols;
  for (int i = 0; i < n; ++i) {   // every argument is checked before the first launch
    FP8T_TRY(check_hp(dy[i], "dy[i]"));
    if (dy[i].rows != x.rows || dy[i].dtype != dy[0].dtype) return fail(FP8_EINVAL, "dy[%d]: rows / dtype differ", i);
    FP8T_TRY(check_cfg(cfg, x.rows, dy[i].cols, x.cols));
    FP8T_TRY(check_ptr(saved[i], "saved[i]"));
    if (dx && dx[i]) FP8T_TRY(check_ptr(dx[i], "dx[i]"));
    if (dw && dw[i]) FP8T_TRY(check_ptr(dw[i], "dw[i]"));
    d.pre[i + 1] = d.pre[i] + dy[i].cols;
    d.nmax = dy[i].cols > d.nmax ? dy[i].cols : d.nmax;
  }
  d.nsum = d.pre[n];
  FP8T_TRY(check_hp(x, "x", gw_hp && dw));
  FP8T_TRY(check_ptr(ws, "ws"));
  const size_t need = shared_ws_bytes(cfg, d, n);
  if (ws_bytes < need) return fail(FP8_EWORKSPACE, "workspace too small (%zu < %zu)", ws_bytes, need);
  const BwdGroupWs gw = carve_bwd_group(cfg, d, n, ws, nullptr);
  cudaStream_t st = S(stream);
  // rowwise with dX and dW for every member: every dY_i's row / column amax by one launch, its
  // row-scaled (dX) and column-scaled (dW) codes by one cast launch
  bool batched = false;
  bool full = dx && dw && dy[0].dtype == FP8_DT_BF16;
  for (int i = 0; full && i < n; ++i) full = dx[i] && dw[i];
  if (group_batchable(cfg, n) && full && knob(KNOB_GROUP_BATCH) == 1) {
    float* am = group_bwd_amax(cfg, d, n, ws);
    FP8T_CUDA(cudaMemsetAsync(am, 0, 4 * group_bwd_amax_floats(cfg, d, n), st), "memset group amax");
    AmaxRCTensor ts[AMAX_RC_MAX];
    CastMulti cm{};
    cm.n = n;
    float* p = am;
    for (int i = 0; i < n; ++i) {
      const BwdWs bi = bwd_member(cfg, gw, d, i);
      float* ar = p;
      float* ac = p + d.M;
      p = ac + dy[i].cols;
      ts[i] = AmaxRCTensor{dy[i].ptr, d.M, dy[i].cols, dy[i].ld, reinterpret_cast<uint32_t*>(ar),
                           reinterpret_cast<uint32_t*>(ac)};
      cm.x[i] = dy[i].ptr; cm.R[i] = d.M; cm.C[i] = dy[i].cols; cm.ld[i] = dy[i].ld;
      cm.amax_q[i] = ar; cm.amax_t[i] = ac;
      cm.q[i] = bi.g; cm.qt[i] = bi.gT;
      cm.scale_q[i] = static_cast<float*>(bi.sg); cm.scale_t[i] = static_cast<float*>(bi.sgT);
    }
    const cudaError_t e = launch_amax_rc(ts, n, 6, st);
    if (e != cudaErrorNotSupported) {
      FP8T_CUDA(e, "group amax dy");
      FP8T_CUDA(launch_cast_dual(cm, true, cfg->fmt_grad, 2, 5, st), "group cast dy");
      batched = true;
    }
  }
  std::vector<GemmProblem> ps;
  for (int i = 0; i < n; ++i) {
    const BwdWs bi = bwd_member(cfg, gw, d, i);
    FP8T_TRY(linear_bwd_impl(cfg, dy[i], nullptr, x, saved[i], nullptr, dx ? dx[i] : nullptr, nullptr,
                             dw ? dw[i] : nullptr, ws, ws_bytes, stream, nullptr, 1, saved[0], dy[0].cols, &bi, &ps,
                             batched));
  }
  return launch_group(ps, st);
}

fp8_status_t fp8_linear_bwd_ex(const fp8_linear_cfg_t* cfg, fp8_hp_t dy, const float* dy_amax, fp8_hp_t x,
                               const void* saved, const fp8_tensor_t* w_fp8, void* dx, float* dx_amax, void* dw,
                               void* ws, size_t ws_bytes, void* stream) {
  return linear_bwd_impl(cfg, dy, dy_amax, x, saved, w_fp8, dx, dx_amax, dw, ws, ws_bytes, stream, nullptr, 1);
}

fp8_status_t fp8_linear_bwd_rs(const fp8_linear_cfg_t* cfg, fp8_hp_t dy, fp8_hp_t x, const void* saved,
                               const fp8_tensor_t* w_fp8, void* dx, fp8_p2p_t rs_win, int nranks, void* dw_shard,
                               void* ws, size_t ws_bytes, void* stream) {
  FP8T_TRY(check_fault());
  if (!rs_win || !dw_shard) return fail(FP8_EINVAL, "rs_win / dw_shard: null");
  if (nranks < 1) return fail(FP8_EINVAL, "nranks < 1");
  if (!cfg || cfg->out_dtype != FP8_DT_BF16) return fail(FP8_EUNSUPPORTED, "fused reduce-scatter: bf16 dW only");
  return linear_bwd_impl(cfg, dy, nullptr, x, saved, w_fp8, dx, nullptr, dw_shard, ws, ws_bytes, stream, rs_win, nranks);
}

static fp8_status_t linear_bwd_impl(const fp8_linear_cfg_t* cfg, fp8_hp_t dy, const float* dy_amax, fp8_hp_t x,
                                    const void* saved, const fp8_tensor_t* w_fp8, void* dx, float* dx_amax, void* dw,
                                    void* ws, size_t ws_bytes, void* stream, fp8_p2p_t rs_win, int rs_nranks,
                                    const void* saved_x, int64_t n_x, const BwdWs* bw_in,
                                    std::vector<GemmProblem>* defer, bool cast_done) {
  FP8T_TRY(check_hp(dy, "dy"));
  const int64_t M = dy.rows, N = dy.cols, K = x.cols;
  const bool gw_hp = cfg && cfg->recipe == FP8_RECIPE_ROWWISE_GW_HP;
  FP8T_TRY(check_hp(x, "x", gw_hp && dw));
  if (x.rows != M) return fail(FP8_EINVAL, "x.rows != dy.rows");
  if (gw_hp && dw && (x.dtype != FP8_DT_BF16 || dy.dtype != FP8_DT_BF16))
    return fail(FP8_EUNSUPPORTED, "rowwise_gw_hp: the BF16 dW GEMM needs bf16 dy and x");
  FP8T_TRY(check_cfg(cfg, M, N, K));
  FP8T_TRY(check_ptr(saved, "saved"));
  FP8T_TRY(check_ptr(ws, "ws"));
  if (dx) FP8T_TRY(check_ptr(dx, "dx"));
  if (dw) FP8T_TRY(check_ptr(dw, "dw"));
  if (!bw_in && ws_bytes < fp8_linear_workspace_bytes(cfg, M, N, K)) return fail(FP8_EWORKSPACE, "workspace too small");
  if (w_fp8) FP8T_TRY(check_w_fp8(cfg, w_fp8, N, K, dx != nullptr));
  if (dy_amax && cfg->recipe != FP8_RECIPE_TENSORWISE)
    return fail(FP8_EUNSUPPORTED, "dy_amax (precomputed tensor amax) needs the tensorwise recipe");
  if (rs_win && (N % ((int64_t)rs_nranks * 256)))
    return fail(FP8_EALIGN, "fused reduce-scatter: N must be a multiple of 256 * nranks");
  const int64_t rs_rows = N / rs_nranks;   // dW rows per rank (FSDP2 dim-0 shard)
  cudaStream_t st = S(stream);
  const bool gb = dy.dtype == FP8_DT_BF16;
  const int ff = cfg->fmt_fwd, fg = cfg->fmt_grad;
  uint32_t* dxam = dx ? reinterpret_cast<uint32_t*>(dx_amax) : nullptr;
  Saved sv = carve_saved(cfg, M, N, K, const_cast<void*>(saved), nullptr);
  if (saved_x) {   // shared-input group: X's backward operand lives in the first member's buffer
    const Saved s0 = carve_saved(cfg, M, n_x, K, const_cast<void*>(saved_x), nullptr);
    sv.xT = s0.xT;
    sv.sx = s0.sx;
  }
  // bw_in: a shared-input group's slice for this member (its dY operands stay until the group's GEMMs)
  BwdWs bw = bw_in ? *bw_in : carve_bwd(cfg, M, N, ws, nullptr);
  const int of32 = cfg->out_dtype == FP8_DT_F32;
  int mode;
  if (cfg->recipe == FP8_RECIPE_TENSORWISE) {
    mode = 0;
    if (!dy_amax) {
      FP8T_CUDA(cudaMemsetAsync(bw.amax, 0, 4, st), "memset");
      FP8T_CUDA(launch_amax(dy.ptr, gb, M, N, dy.ld, 1, (uint32_t*)bw.amax, nullptr, nullptr, st), "amax dy");
    }
    const float* agp = dy_amax ? dy_amax : bw.amax;
    FP8T_CUDA(launch_cast(dy.ptr, gb, fg, M, N, dy.ld, 1, 0, agp, agp, bw.g, nullptr, (float*)bw.sg, nullptr, st),
              "cast dy");
  } else if (cfg->recipe == FP8_RECIPE_ROWWISE || gw_hp) {
    mode = 1;
    float* ar = bw.amax;
    float* ac = ar + M;
    const bool colcopy = dw && !gw_hp;   // gw_hp: dW is a BF16 GEMM on the hp dY
    if (cast_done) goto gemms;           // a shared-input group cast every member's dY by one launch pair
    if (!dx && !colcopy) goto gemms;
    FP8T_CUDA(cudaMemsetAsync(bw.amax, 0, 4 * (M + N), st), "memset");
    FP8T_CUDA(launch_amax(dy.ptr, gb, M, N, dy.ld, colcopy ? (dx ? 6 : 4) : 2, nullptr, (uint32_t*)ar,
                          (uint32_t*)ac, st),
              "amax dy");
    FP8T_CUDA(launch_cast(dy.ptr, gb, fg, M, N, dy.ld, dx ? 2 : 0, colcopy ? 5 : 0, ar, ac, bw.g, bw.gT,
                          (float*)bw.sg, (float*)bw.sgT, st),
              "cast dy");
  } else {
    mode = 2;
    FP8T_CUDA(launch_mx_cast(dy.ptr, gb, fg, cfg->mx_round == FP8_MX_RCEIL, M, N, dy.ld, dx ? bw.g : nullptr,
                             (uint8_t*)bw.sg, dw ? bw.gT : nullptr, (uint8_t*)bw.sgT, st, mx_transposed()),
              "mx cast dy");
  }
gemms:
  if (!dx && !dw) return FP8_OK;
  // zeroed after the dY cast has read dy_amax, so the two may share a buffer
  if (dxam) FP8T_CUDA(cudaMemsetAsync(dxam, 0, 4, st), "memset dx_amax");
  if (gw_hp) {
    // dX in FP8 (row-scaled dY x column-scaled W, read MN-major); dW = dY^T X in BF16 on the
    // high-precision operands (both row-major [M, .] -> MN-major)
    if (dx) {
      GemmProblem p{bw.g, sv.wT, fg, ff, 0, 1, bw.sg, sv.sw, 1, M, K, N, N, K, dx, of32, K, 0, dxam};
      if (defer) defer->push_back(p);
      else FP8T_CUDA(launch_gemm(p, st), "gemm dx");
    }
    if (dw) {
      GemmProblem p{static_cast<const uint8_t*>(dy.ptr), static_cast<const uint8_t*>(x.ptr), 0, 0, 1, 1, nullptr,
                    nullptr, 0, N, K, M, dy.ld, x.ld, dw, of32, K, 1};
      if (defer) {
        defer->push_back(p);
        return FP8_OK;
      }
      if (rs_win) FP8T_TRY(p2p_rs_begin(rs_win, rs_rows, K, st, p));
      FP8T_CUDA(launch_gemm(p, st), "gemm dw bf16");
      if (rs_win) FP8T_TRY(p2p_rs_end(rs_win, rs_rows, K, dw, K, st));
    }
    return FP8_OK;
  }
  // dX and dW run as one persistent launch (tiles of dX, then dW): no wave tail between them
  GemmProblem ps[2];
  int n = 0;
  if (mode == 0) {
    // tensorwise: operands are the row-major codes; B of dX and both operands of dW are MN-major
    const uint8_t* wq = w_fp8 ? w_fp8->q : sv.wT;
    // dX[M,K] = dY[M,N] . W[N,K]: A = Gq K-major over N, B = Wq stored [N,K] = MN-major
    if (dx) ps[n++] = GemmProblem{bw.g, wq, fg, ff, 0, 1, bw.sg, sv.sw, 0, M, K, N, N, K, dx, of32, K, 0, dxam};
    // dW[N,K] = dY^T . X: A = Gq stored [M,N] = MN-major, B = Xq stored [M,K] = MN-major
    if (dw) ps[n++] = GemmProblem{bw.g, sv.xT, fg, ff, 1, 1, bw.sg, sv.sx, 0, N, K, M, N, K, dw, of32, K};
  } else if (mode == 1) {
    // rowwise: column-scaled copies are row-major too -> read MN-major
    // dX[M,K] = dY_r[M,N] . W_c[N,K]: A K-major over N, B stored [N,K] = MN-major
    if (dx) ps[n++] = GemmProblem{bw.g, sv.wT, fg, ff, 0, 1, bw.sg, sv.sw, mode, M, K, N, N, K, dx, of32, K, 0, dxam};
    // dW[N,K] = dY_c^T . X_c: A stored [M,N] = MN-major, B stored [M,K] = MN-major
    if (dw) ps[n++] = GemmProblem{bw.gT, sv.xT, fg, ff, 1, 1, bw.sgT, sv.sx, mode, N, K, M, N, K, dw, of32, K};
  } else if (!mx_transposed()) {
    const uint8_t* w1 = w_fp8 ? w_fp8->q_t : sv.wT;
    const void* s1 = w_fp8 ? w_fp8->scale_t : sv.sw;
    // MXFP8: dim1 copies (blocks along the contraction dim) kept in the input's row-major layout
    // and read MN-major, like the tensorwise / rowwise backward
    // dX[M,K] = dY[M,N] . W : A = dY dim0 (K-major over N), B = W dim1 stored [N,K] = MN-major
    if (dx) ps[n++] = GemmProblem{bw.g, w1, fg, ff, 0, 1, bw.sg, s1, mode, M, K, N, N, K, dx, of32, K, 0, dxam};
    // dW[N,K] = dY^T . X : A = dY dim1 stored [M,N] = MN-major, B = X dim1 stored [M,K] = MN-major
    if (dw) ps[n++] = GemmProblem{bw.gT, sv.xT, fg, ff, 1, 1, bw.sgT, sv.sx, mode, N, K, M, N, K, dw, of32, K};
  } else {
    const uint8_t* w1 = w_fp8 ? w_fp8->q_t : sv.wT;
    const void* s1 = w_fp8 ? w_fp8->scale_t : sv.sw;
    // MXFP8 with transposed dim1 copies (knob mx_transposed = 1), all operands K-major
    // dX[M,K] = dY[M,N] . W  : A = dY (K-major over N), B = W^T [K,N]
    if (dx) ps[n++] = GemmProblem{bw.g, w1, fg, ff, 0, 0, bw.sg, s1, mode, M, K, N, N, N, dx, of32, K, 0, dxam};
    // dW[N,K] = dY^T[N,M] . X : A = dY^T [N,M], B = X^T [K,M]
    if (dw) ps[n++] = GemmProblem{bw.gT, sv.xT, fg, ff, 0, 0, bw.sgT, sv.sx, mode, N, K, M, M, M, dw, of32, K};
  }
  if (defer) {
    defer->insert(defer->end(), ps, ps + n);
    return FP8_OK;
  }
  if (rs_win && dw) FP8T_TRY(p2p_rs_begin(rs_win, rs_rows, K, st, ps[n - 1]));   // dW is the last problem
  FP8T_CUDA(launch_gemms(ps, n, st), "gemm dx/dw");
  if (rs_win && dw) FP8T_TRY(p2p_rs_end(rs_win, rs_rows, K, dw, K, st));
  return FP8_OK;
}

// ---------------------------------------------------------------------------
// MoE scaled grouped GEMM (PAPER.md:739 scaled_grouped_mm; reading R-c22): the Float8Linear
// recipe per expert on expert-sorted tokens.  One M-grouped launch for Y; one launch carrying
// the M-grouped dX and the K-grouped dW problems.  Scaling units never cross an expert: rowwise
// column scales are kept per (expert, column) (segmented amax / cast kernels).
// ---------------------------------------------------------------------------
}  // extern "C"

namespace {

struct GSaved {
  uint8_t* xT; uint8_t* wT;   // tensorwise: Xq [T,K], Wq [E*N,K]; rowwise: per-expert column-scaled copies
  float* sx; float* sw;       // tensorwise [1], [1]; rowwise [E*K], [E*K]
};
GSaved carve_gsaved(const fp8_linear_cfg_t* cfg, int64_t T, int64_t E, int64_t N, int64_t K, void* base,
                    size_t* bytes) {
  Carve c(base);
  GSaved g;
  g.xT = c.take<uint8_t>((size_t)T * K);
  g.wT = c.take<uint8_t>((size_t)E * N * K);
  const bool tw = cfg->recipe == FP8_RECIPE_TENSORWISE;
  g.sx = c.take<float>(tw ? 4 : 4 * E * K);
  g.sw = c.take<float>(tw ? 4 : 4 * E * K);
  if (bytes) *bytes = c.off;
  return g;
}
struct GFwdWs {
  uint8_t* xq; uint8_t* wq;          // rowwise row-scaled codes
  float* amax;                       // tensorwise [2]; rowwise [T + E*K + E*N + E*K]
  float* sxr; float* swr;            // rowwise row scales [T], [E*N]
};
GFwdWs carve_gfwd(const fp8_linear_cfg_t* cfg, int64_t T, int64_t E, int64_t N, int64_t K, void* base, size_t* bytes) {
  Carve c(base);
  GFwdWs w{};
  if (cfg->recipe == FP8_RECIPE_TENSORWISE) {
    w.amax = c.take<float>(8);
  } else {
    w.xq = c.take<uint8_t>((size_t)T * K);
    w.wq = c.take<uint8_t>((size_t)E * N * K);
    w.amax = c.take<float>(4 * (T + E * K + E * N + E * K));
    w.sxr = c.take<float>(4 * T);
    w.swr = c.take<float>(4 * E * N);
  }
  if (bytes) *bytes = c.off;
  return w;
}
struct GBwdWs {
  uint8_t* g; uint8_t* gT;           // dY row-scaled [T,N]; rowwise: per-expert column-scaled [T,N]
  float* amax;                       // tensorwise [1]; rowwise [T + E*N]
  float* sg; float* sgT;             // tensorwise [1]; rowwise [T], [E*N]
};
GBwdWs carve_gbwd(const fp8_linear_cfg_t* cfg, int64_t T, int64_t E, int64_t N, void* base, size_t* bytes) {
  Carve c(base);
  GBwdWs w{};
  const bool tw = cfg->recipe == FP8_RECIPE_TENSORWISE;
  w.g = c.take<uint8_t>((size_t)T * N);
  w.gT = tw ? nullptr : c.take<uint8_t>((size_t)T * N);
  w.amax = c.take<float>(tw ? 4 : 4 * (T + E * N));
  w.sg = c.take<float>(tw ? 4 : 4 * T);
  w.sgT = tw ? w.sg : c.take<float>(4 * E * N);
  if (bytes) *bytes = c.off;
  return w;
}

fp8_status_t check_grouped(const fp8_linear_cfg_t* cfg, int64_t T, int64_t E, int64_t N, int64_t K, const int* offs) {
  FP8T_TRY(check_fault());
  if (!cfg) return fail(FP8_EINVAL, "cfg: null pointer");
  if (cfg->recipe != FP8_RECIPE_TENSORWISE && cfg->recipe != FP8_RECIPE_ROWWISE)
    return fail(FP8_EUNSUPPORTED, "grouped GEMM: tensorwise or rowwise recipe");
  FP8T_TRY(check_fmt(cfg->fmt_fwd));
  FP8T_TRY(check_fmt(cfg->fmt_grad));
  if (cfg->out_dtype != FP8_DT_BF16 && cfg->out_dtype != FP8_DT_F32) return fail(FP8_EINVAL, "bad out_dtype");
  if (E < 1 || E > GEMM_MAX_GROUPS) return fail(FP8_EINVAL, "E must be in [1, %d]", GEMM_MAX_GROUPS);
  if (!offs) return fail(FP8_EINVAL, "offs: null pointer");
  if (T < 128 || T % 128) return fail(FP8_EALIGN, "T (tokens) must be a positive multiple of 128");
  if (N < 128 || N % 128) return fail(FP8_EALIGN, "N (expert rows) must be a positive multiple of 128");
  if (K < 16 || K % 16) return fail(FP8_EALIGN, "K must be a positive multiple of 16");
  if (T > (1 << 30) || E * N > (1 << 30)) return fail(FP8_EINVAL, "dims too large");
  return FP8_OK;
}

}  // namespace

extern "C" {

size_t fp8_grouped_saved_bytes(const fp8_linear_cfg_t* cfg, int64_t T, int64_t E, int64_t N, int64_t K) {
  if (!cfg) return 0;
  size_t b = 0;
  carve_gsaved(cfg, T, E, N, K, nullptr, &b);
  return b;
}

size_t fp8_grouped_workspace_bytes(const fp8_linear_cfg_t* cfg, int64_t T, int64_t E, int64_t N, int64_t K) {
  if (!cfg) return 0;
  size_t f = 0, b = 0;
  carve_gfwd(cfg, T, E, N, K, nullptr, &f);
  carve_gbwd(cfg, T, E, N, nullptr, &b);
  return f > b ? f : b;
}

fp8_status_t fp8_grouped_linear_fwd(const fp8_linear_cfg_t* cfg, fp8_hp_t x, fp8_hp_t w, int64_t E, const int32_t* offs,
                                    void* y, void* saved, void* ws, size_t ws_bytes, void* stream) {
  FP8T_TRY(check_hp(x, "x"));
  FP8T_TRY(check_hp(w, "w"));
  const int64_t T = x.rows, K = x.cols;
  if (E < 1 || w.rows % E) return fail(FP8_EINVAL, "w.rows must be E * N");
  const int64_t N = w.rows / E;
  if (w.cols != K) return fail(FP8_EINVAL, "w.cols != x.cols");
  FP8T_TRY(check_grouped(cfg, T, E, N, K, offs));
  FP8T_TRY(check_ptr(y, "y"));
  FP8T_TRY(check_ptr(saved, "saved"));
  FP8T_TRY(check_ptr(ws, "ws"));
  if (ws_bytes < fp8_grouped_workspace_bytes(cfg, T, E, N, K)) return fail(FP8_EWORKSPACE, "workspace too small");
  cudaStream_t st = S(stream);
  const bool xb = x.dtype == FP8_DT_BF16, wb = w.dtype == FP8_DT_BF16;
  const int ff = cfg->fmt_fwd, of32 = cfg->out_dtype == FP8_DT_F32;
  GSaved sv = carve_gsaved(cfg, T, E, N, K, saved, nullptr);
  GFwdWs fw = carve_gfwd(cfg, T, E, N, K, ws, nullptr);
  Seg tok{offs, (int)E, 0}, exp_rows{nullptr, 0, (int)N};
  GemmProblem p{};
  if (cfg->recipe == FP8_RECIPE_TENSORWISE) {
    uint32_t* a = reinterpret_cast<uint32_t*>(fw.amax);
    FP8T_CUDA(cudaMemsetAsync(a, 0, 8, st), "memset");
    FP8T_CUDA(launch_amax(x.ptr, xb, T, K, x.ld, 1, a, nullptr, nullptr, st), "amax x");
    FP8T_CUDA(launch_amax(w.ptr, wb, E * N, K, w.ld, 1, a + 1, nullptr, nullptr, st), "amax w");
    FP8T_CUDA(launch_cast(x.ptr, xb, ff, T, K, x.ld, 1, 0, fw.amax, fw.amax, sv.xT, nullptr, sv.sx, nullptr, st), "cast x");
    FP8T_CUDA(launch_cast(w.ptr, wb, ff, E * N, K, w.ld, 1, 0, fw.amax + 1, fw.amax + 1, sv.wT, nullptr, sv.sw, nullptr,
                          st), "cast w");
    p = GemmProblem{sv.xT, sv.wT, ff, ff, 0, 0, sv.sx, sv.sw, 0, T, N, K, K, K, y, of32, N};
  } else {
    float* axr = fw.amax;
    float* axc = axr + T;          // [E, K] per (expert, column) over the expert's tokens
    float* awr = axc + E * K;      // [E*N]
    float* awc = awr + E * N;      // [E, K] per (expert, column) over the expert's N rows
    FP8T_CUDA(cudaMemsetAsync(fw.amax, 0, 4 * (T + E * K + E * N + E * K), st), "memset");
    FP8T_CUDA(launch_amax(x.ptr, xb, T, K, x.ld, 6, nullptr, (uint32_t*)axr, (uint32_t*)axc, st, tok), "amax x");
    FP8T_CUDA(launch_amax(w.ptr, wb, E * N, K, w.ld, 6, nullptr, (uint32_t*)awr, (uint32_t*)awc, st, exp_rows),
              "amax w");
    FP8T_CUDA(launch_cast(x.ptr, xb, ff, T, K, x.ld, 2, 5, axr, axc, fw.xq, sv.xT, fw.sxr, sv.sx, st, tok), "cast x");
    FP8T_CUDA(launch_cast(w.ptr, wb, ff, E * N, K, w.ld, 2, 5, awr, awc, fw.wq, sv.wT, fw.swr, sv.sw, st, exp_rows),
              "cast w");
    p = GemmProblem{fw.xq, fw.wq, ff, ff, 0, 0, fw.sxr, fw.swr, 1, T, N, K, K, K, y, of32, N};
  }
  p.grouped = 1;
  p.G = (int)E;
  p.offs = offs;
  FP8T_CUDA(launch_gemm(p, st), "grouped gemm fwd");
  return FP8_OK;
}

fp8_status_t fp8_grouped_linear_bwd(const fp8_linear_cfg_t* cfg, fp8_hp_t dy, fp8_hp_t x, int64_t E, const int32_t* offs,
                                    const void* saved, void* dx, void* dw, void* ws, size_t ws_bytes, void* stream) {
  FP8T_TRY(check_hp(dy, "dy"));
  FP8T_TRY(check_hp(x, "x", false));
  const int64_t T = dy.rows, N = dy.cols, K = x.cols;
  if (x.rows != T) return fail(FP8_EINVAL, "x.rows != dy.rows");
  FP8T_TRY(check_grouped(cfg, T, E, N, K, offs));
  FP8T_TRY(check_ptr(saved, "saved"));
  FP8T_TRY(check_ptr(ws, "ws"));
  if (dx) FP8T_TRY(check_ptr(dx, "dx"));
  if (dw) FP8T_TRY(check_ptr(dw, "dw"));
  if (ws_bytes < fp8_grouped_workspace_bytes(cfg, T, E, N, K)) return fail(FP8_EWORKSPACE, "workspace too small");
  if (!dx && !dw) return FP8_OK;
  cudaStream_t st = S(stream);
  const bool gb = dy.dtype == FP8_DT_BF16;
  const int ff = cfg->fmt_fwd, fg = cfg->fmt_grad, of32 = cfg->out_dtype == FP8_DT_F32;
  GSaved sv = carve_gsaved(cfg, T, E, N, K, const_cast<void*>(saved), nullptr);
  GBwdWs bw = carve_gbwd(cfg, T, E, N, ws, nullptr);
  Seg tok{offs, (int)E, 0};
  GemmProblem ps[2];
  int n = 0;
  if (cfg->recipe == FP8_RECIPE_TENSORWISE) {
    FP8T_CUDA(cudaMemsetAsync(bw.amax, 0, 4, st), "memset");
    FP8T_CUDA(launch_amax(dy.ptr, gb, T, N, dy.ld, 1, (uint32_t*)bw.amax, nullptr, nullptr, st), "amax dy");
    FP8T_CUDA(launch_cast(dy.ptr, gb, fg, T, N, dy.ld, 1, 0, bw.amax, bw.amax, bw.g, nullptr, bw.sg, nullptr, st),
              "cast dy");
    // dX_g = dY_g W_g: A = Gq K-major over N; B = Wq [E*N, K] read MN-major (expert g = contraction rows g*N..)
    if (dx) ps[n++] = GemmProblem{bw.g, sv.wT, fg, ff, 0, 1, bw.sg, sv.sw, 0, T, K, N, N, K, dx, of32, K};
    // dW_g = dY_g^T X_g: both MN-major, contraction over the expert's tokens
    if (dw) ps[n++] = GemmProblem{bw.g, sv.xT, fg, ff, 1, 1, bw.sg, sv.sx, 0, N, K, T, N, K, dw, of32, K};
  } else {
    float* ar = bw.amax;
    float* ac = ar + T;   // [E, N]
    FP8T_CUDA(cudaMemsetAsync(bw.amax, 0, 4 * (T + E * N), st), "memset");
    FP8T_CUDA(launch_amax(dy.ptr, gb, T, N, dy.ld, dw ? (dx ? 6 : 4) : 2, nullptr, (uint32_t*)ar, (uint32_t*)ac, st, tok),
              "amax dy");
    FP8T_CUDA(launch_cast(dy.ptr, gb, fg, T, N, dy.ld, dx ? 2 : 0, dw ? 5 : 0, ar, ac, bw.g, bw.gT, bw.sg, bw.sgT, st,
                          tok),
              "cast dy");
    if (dx) ps[n++] = GemmProblem{bw.g, sv.wT, fg, ff, 0, 1, bw.sg, sv.sw, 1, T, K, N, N, K, dx, of32, K};
    if (dw) ps[n++] = GemmProblem{bw.gT, sv.xT, fg, ff, 1, 1, bw.sgT, sv.sx, 1, N, K, T, N, K, dw, of32, K};
  }
  for (int i = 0; i < n; ++i) {
    ps[i].grouped = ps[i].a_mn && ps[i].b_mn ? 2 : 1;
    ps[i].G = (int)E;
    ps[i].offs = offs;
  }
  FP8T_CUDA(launch_gemms(ps, n, st), "grouped gemm dx/dw");
  return FP8_OK;
}

}  // extern "C"
