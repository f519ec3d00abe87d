// Internal launcher declarations (not part of the C-ABI).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <mutex>

namespace fp8t {

void count_launch();

// ---- kernel-variant knobs (fp8_set_knob / fp8_get_knob) ----
// The defaults are the product path; the other values are A/B variants the tests and tools/
// select explicitly.  Read with relaxed atomics on the host per launch -- never from the process
// environment, so results cannot depend on the caller's environment.
enum Knob {
  KNOB_AMAX_TILE_TMA = 0,   // 1: TMA-ring row/col amax strip kernel; 0: register-only tile kernel
  KNOB_CAST_GRID,           // >0: cap the persistent cast / amax / MX grids (tests: many tiles per CTA)
  KNOB_AMAX_BLOCKS_PER_SM,  // flat tensorwise amax: resident CTAs per SM (1..9)
  KNOB_AMAX_LOADS,          // flat tensorwise amax: 16-byte loads in flight per thread (4, 8, 12, 16)
  KNOB_MX_CAST_TMA,         // 1: TMA-ring MX cast (bf16); 0: register-only MX cast
  KNOB_GEMM_CTA_GROUP,      // 2: CTA-pair tcgen05 tiles; 1: single-CTA tiles
  KNOB_GEMM_DEBUG,          // tools/gemm_bench.py pipeline-isolation modes (0 = off)
  KNOB_GEMM_SCHED,          // 1: dynamic tile scheduler; 0: static round-robin tiles
  KNOB_MX_SF_SPLIT,         // MX GEMM scale-factor copier split (1 = default)
  KNOB_GEMM_RASTER,         // <0: per-problem raster (choose_raster); >=0: fixed group width for all
  KNOB_MX_N192,             // 1: MX GEMM with N = 192 tiles, double-buffered accumulators
  KNOB_GEMM_STAGES,         // 3: 3 stages x 2 K atoms; 4 / 6: 4 / 6 stages x 1 atom
  KNOB_GEMM_EPI,            // 0: epilogue warps by K (8 for K <= 1024, else 4); 4 / 8: forced
  KNOB_MX_TRANSPOSED,       // 1: MX dim1 copies written transposed, read K-major (fwd and bwd must agree)
  KNOB_TW_DUAL,             // 1: tensorwise forward X/W amax and cast by one launch each; 0: four launches
  KNOB_GEMM_KSERP,          // 1: odd waves of GEMM tiles walk K backwards (L2 reuse across waves); 0: all forward
  KNOB_GEMM_N512,           // 1: plain FP8 GEMMs with every N % 512 == 0 use 256 x 512 CTA-pair tiles (2: auto, K >= 8192)
  KNOB_GEMM_L2PF,           // >0: the GEMM producer prefetches operand boxes this many stages ahead into L2
  KNOB_MX_CAST_OCC3,        // 1: MX cast (dim0 + dim1, row-major dim1) with a 2-deep ring at 3 CTAs per SM
  KNOB_AMAX_BULK,           // 1: tensorwise amax of contiguous tensors through 1-D bulk copies into a smem ring
  KNOB_AMAX_RC,             // 1: row / column amax by amax_rc_kernel (no CTA barrier per tile, multi-tensor)
  KNOB_AMAX_RC_DEBUG,       // A/B only: bit 0 consumers skip the tile (results invalid)
  KNOB_GROUP_BATCH,         // 1: a rowwise shared-input group's amax / cast launches batched over X + every W_i (fwd), every dY_i (bwd)
  KNOB_MX_CAST_DEBUG,       // A/B only: bit 0 the MX TMA cast skips its code stores (results invalid)
  KNOB_MX_CAST_WS,          // 1: bf16 MX casts with row-major dim1 copies by the warp-specialised kernel (0: the ring kernel)
  KNOB_GEMM_ST_EF,          // 1: GEMM bf16 outputs stored with an L2 evict-first hint
  KNOB_WAIT_SLEEP,          // barrier waits with a suspend-time hint: bit 0 amax_rc / MX ws casts, bit 1 GEMM epilogue,
                            // bit 2 GEMM producer, bit 3 GEMM MMA + SF copier
  KNOB_GEMM_L2HINT,         // A/B: L2 eviction hints on the GEMM operand loads (1 A evict_last, 2 + B evict_first, 3 + B normal)
  KNOB_GEMM_AFILL,          // 1: 256 x 512 tiles: per K step both N halves' MMAs, A kept in the tensor core's collector
  KNOB_MX_CAST_TSTORE,      // 1 (default): the MX ring cast (dim0 + row-major dim1) writes its codes by TMA tensor stores
  KNOB_CAST_RC_TMA,         // rowwise casts of bf16 128-multiple tensors by the TMA-ring kernel with TMA stores: 1 auto (<= 12288 tiles), 2 always
  KNOB_CAST_RC_WIDE,        // A/B: the rowwise TMA cast as 1 CTA of 512 threads per SM with a 5-deep ring
  KNOB_GEMM_EPI_TMA,        // 1: 256-wide GEMM tiles with bf16 outputs store them by TMA (one 2 KB chunk buffer per warp)
  KNOB_WATCHDOG_MS,         // peer waits (P2P gather, fused reduce-scatter, async-TP) give up after this many ms
                            // and report FP8_ECUDA at the next call; 0 = wait forever
  KNOB_COUNT
};
int knob(Knob k);

// ---- asynchronous device faults (instead of trap) ----
// A kernel that gives up waiting on a peer (watchdog) or rejects device-side arguments writes a code to
// the process-wide fault word -- pinned host memory mapped into every device -- and returns without
// trapping, so the CUDA context survives.  The next ABI call that checks it (fp8_check_async_error and
// every P2P / FSDP / grouped / async-TP entry point) reports it as a status and clears it.
enum FaultCode : unsigned {
  FAULT_P2P_AMAX_WAIT = 1,   // a peer's amax signal never arrived (peer = slot, low bits = epoch)
  FAULT_P2P_DONE_WAIT = 2,   // a peer's pushes / reduce-scatter tiles never completed
  FAULT_TP_CHUNK_WAIT = 3,   // async-TP: a chunk of A rows never arrived
  FAULT_GROUP_OFFSETS = 4,   // grouped GEMM: device offsets not 0 = o0 <= ... <= oG = extent, multiples of 128
};
__host__ __device__ constexpr unsigned fault_pack(unsigned code, unsigned peer, unsigned epoch) {
  return (code << 24) | ((peer & 0xFFu) << 16) | (epoch & 0xFFFFu);
}
// Device-visible pointer to the fault word (nullptr if the pinned allocation failed: then the kernels
// fall back to waiting without a watchdog); watchdog timeout in ns (knob watchdog_ms; 0 = none).
unsigned* fault_word(cudaStream_t st = nullptr);   // st: not allocated while st is capturing
unsigned long long watchdog_ns();

// Multiprocessor count of the current device (cached per device).
int device_sm_count();
// Once per (kernel, device): raise the dynamic shared-memory limit of `Kern` to `bytes`.  The
// attribute is per device context, so a process driving several GPUs sets it on each.
constexpr int MAX_DEVICES = 64;
cudaError_t current_device(int* dev);
template <auto Kern>
cudaError_t ensure_smem(int bytes) {
  static std::once_flag flags[MAX_DEVICES];
  static cudaError_t errs[MAX_DEVICES];
  int dev = 0;
  cudaError_t e = current_device(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= MAX_DEVICES) return cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  std::call_once(flags[dev], [&] { errs[dev] = cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); });
  return errs[dev];
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (nullptr if unavailable).
PFN_cuTensorMapEncodeTiled_v12000 get_encode();

// Launch accounting + optional per-launch CUDA-event timing (fp8_profile_enable).
enum { K_AMAX = 0, K_CAST = 1, K_MX = 2, K_TRANSPOSE = 3, K_GEMM = 4, K_GEMM_MX = 5, K_GEMM_BF16 = 6,
       K_SYNC = 7 };   // K_SYNC: the P2P gather's signal / wait kernels
struct LaunchScope {
  int slot;
  cudaStream_t st;
  LaunchScope(int kind, cudaStream_t s);
  ~LaunchScope();
};

// Row segments for the grouped (MoE) recipe: column amaxes / column scales are kept per segment,
// out index = segment(row) * C + col.  offs (device, G+1 non-decreasing row offsets, multiples of
// 128) or a fixed seg_rows (multiple of 128); neither = one segment (the plain column scales).
struct Seg {
  const int* offs = nullptr;
  int G = 0;
  int seg_rows = 0;
};
// amax_tile: mode bit0 tensor -> at[1], bit1 rows -> ar[R], bit2 cols -> ac[C] (u32 |x| bits, pre-zeroed)
cudaError_t launch_amax(const void* x, bool bf16, int64_t R, int64_t C, int64_t ld, int mode, uint32_t* at,
                        uint32_t* ar, uint32_t* ac, cudaStream_t st, const Seg& seg = Seg{});
// cast_tile: scale modes 0 none / 1 tensor / 2 row / 3 col for q (row-major) and qt (transposed);
// tm = 5: column-scaled second copy written row-major (MN-major operand of the rowwise backward)
cudaError_t launch_cast(const void* x, bool bf16, int fmt, int64_t R, int64_t C, int64_t ld, int qm, int tm,
                        const float* aq, const float* at, uint8_t* q, uint8_t* qt, float* sq, float* st,
                        cudaStream_t s, const Seg& seg = Seg{});
// Row (mode 2) / column (4) / row+column (6) amax of two bf16 tensors in one launch (outputs pre-zeroed);
// cudaErrorNotSupported if a shape is not a multiple of 128 (launch them separately then).
cudaError_t launch_amax_dual(const void* x0, int64_t R0, int64_t C0, int64_t ld0, const void* x1, int64_t R1, int64_t C1,
                             int64_t ld1, int mode, uint32_t* ar0, uint32_t* ac0, uint32_t* ar1, uint32_t* ac1,
                             cudaStream_t st);
// Tensorwise amax of two contiguous tensors (same dtype) in one launch; outputs pre-zeroed.
// Row (mode 2) / column (4) / row+column (6) amax of up to AMAX_RC_MAX bf16 tensors in one launch
// (amax_rc_kernel); outputs pre-zeroed; cudaErrorNotSupported if a shape does not fit the TMA path.
constexpr int AMAX_RC_MAX = 9;   // X + FP8_SHARED_MAX weights
struct AmaxRCTensor {
  const void* x;
  int64_t R, C, ld;
  uint32_t* row;   // [R] (mode & 2)
  uint32_t* col;   // [C] (mode & 4; [G][C] for tensor 0 with a Seg)
};
struct AmaxRCArgs {
  CUtensorMap map[AMAX_RC_MAX];
  int n;
  int tstart[AMAX_RC_MAX + 1];
  int tiles_x[AMAX_RC_MAX];
  int strip0[AMAX_RC_MAX];
  int64_t C[AMAX_RC_MAX];
  uint32_t* row[AMAX_RC_MAX];
  uint32_t* col[AMAX_RC_MAX];
  Seg seg;
  int dbg;   // knob amax_rc_debug (A/B experiments only)
  int sleep; // knob wait_sleep bit 0: barrier waits sleep instead of spinning
};
cudaError_t launch_amax_rc(const AmaxRCTensor* ts, int n, int mode, cudaStream_t st, const Seg& seg = Seg{});
cudaError_t launch_amax_flat_dual(const void* x0, int64_t n0_elems, uint32_t* out0, const void* x1, int64_t n1_elems,
                                  uint32_t* out1, bool bf16, cudaStream_t st);
// Two tensors (same format and scale modes) cast by one launch; tiles[] is filled by the launcher.
// Up to CAST_MULTI_MAX tensors (same format and scale modes) cast by one launch: tensor k's tiles follow
// tensor k-1's; n = 0 is read as 2 (the forward's X and W); tstart[] is filled by the launcher.
constexpr int CAST_MULTI_MAX = 9;
struct CastMulti {
  const void* x[CAST_MULTI_MAX];
  int64_t R[CAST_MULTI_MAX], C[CAST_MULTI_MAX], ld[CAST_MULTI_MAX];
  const float* amax_q[CAST_MULTI_MAX];
  const float* amax_t[CAST_MULTI_MAX];
  uint8_t* q[CAST_MULTI_MAX];
  uint8_t* qt[CAST_MULTI_MAX];
  float* scale_q[CAST_MULTI_MAX];
  float* scale_t[CAST_MULTI_MAX];
  int n;
  int tstart[CAST_MULTI_MAX + 1];
};
using CastDual = CastMulti;
// Rowwise casts (row-scaled codes + column-scaled codes, both row-major) of up to CAST_MULTI_MAX bf16 tensors by
// the persistent TMA kernel (TMA loads and stores); filled by launch_cast_dual / launch_cast.
struct CastRCArgs {
  CUtensorMap in[CAST_MULTI_MAX];   // bf16 [R, C], 128 x 128 boxes
  CUtensorMap oq[CAST_MULTI_MAX];   // u8 [R, C] row-scaled codes
  CUtensorMap ot[CAST_MULTI_MAX];   // u8 [R, C] column-scaled codes
  int n;
  int tstart[CAST_MULTI_MAX + 1];
  int tiles_x[CAST_MULTI_MAX];
  const float* amax_q[CAST_MULTI_MAX];
  const float* amax_t[CAST_MULTI_MAX];
  float* scale_q[CAST_MULTI_MAX];
  float* scale_t[CAST_MULTI_MAX];
};
cudaError_t launch_cast_dual(CastMulti a, bool bf16, int fmt, int qm, int tm, cudaStream_t s);
// Tensorwise amax of n <= AMAX_MULTI_MAX tensors in one launch; out[t] (u32 bit patterns of
// non-negative floats) must be zeroed by the caller.  chunk_start[t] = first warp chunk of
// tensor t (chunks of 256 16-byte vectors within one row), chunk_start[n] = total.
constexpr int AMAX_MULTI_MAX = 48;
struct AmaxMultiArgs {
  int n;
  const uint8_t* ptr[AMAX_MULTI_MAX];
  int64_t ld_bytes[AMAX_MULTI_MAX];
  int64_t vecs[AMAX_MULTI_MAX];   // 16-byte vectors per row
  int64_t cpr[AMAX_MULTI_MAX];    // chunks per row
  int64_t chunk_start[AMAX_MULTI_MAX + 1];
  uint8_t bf16[AMAX_MULTI_MAX];
  uint32_t* out;
};
cudaError_t launch_amax_multi(const AmaxMultiArgs& a, cudaStream_t st);
// MXFP8 dim0 (q0, sf0) and/or dim1 (q1, sf1) casts, blocked E8M0 layout; tr1: dim1 codes written
// transposed [C,R] (else in the input's layout [R,C])
cudaError_t launch_mx_cast(const void* x, bool bf16, int fmt, bool rceil, int64_t R, int64_t C, int64_t ld,
                           uint8_t* q0, uint8_t* sf0, uint8_t* q1, uint8_t* sf1, cudaStream_t s, bool tr1 = true);
// Rank-major gathered dim1 E8M0 tiles [P][Kt][Tl][512 B] -> blocked full layout [Kt][P*Tl][512 B].
cudaError_t launch_sf_unshard(const uint8_t* in, int P, int64_t Kt, int64_t Tl, uint8_t* out, cudaStream_t s);
// ---- fused FP8 FSDP gather over NVLink peer memory (p2p.cu, cast_push in cast_kernels.cu) ----
constexpr int P2P_MAXP = 64;
struct P2PSig {                        // tail of every rank's window, written by peers
  unsigned long long amax[P2P_MAXP];   // slot p: (epoch << 32) | amax bits of rank p's shard
  unsigned long long done[P2P_MAXP];   // slot p: last epoch whose pushes from rank p are visible
  unsigned int ctas;                   // local: finished CTAs of the running cast_push (last-CTA ticket)
  unsigned int rs_cnt[P2P_MAXP];       // local: finished epilogue warps per D row chunk (fused reduce-scatter)
  float scratch[4];                    // local: [0] = 0 (barrier payload), [1..2] barrier scale / amax sink
};
struct P2PPeers {
  uint8_t* buf[P2P_MAXP];              // every rank's gather buffer (peer pointers, UVA)
  P2PSig* sig[P2P_MAXP];
  int P, rank;
};
// Tensorwise cast of the shard x [R, C] with the device scale *scale, every 8-byte code group
// stored to all P gather buffers at byte offset slot_off (rank-rotated order); the last CTA then
// publishes `epoch` in done[rank] of every peer (release, system scope).
cudaError_t launch_cast_push(const void* x, bool bf16, int fmt, int64_t R, int64_t C, int64_t ld, const float* scale,
                             const P2PPeers& pe, int64_t slot_off, P2PSig* mine, uint32_t epoch, cudaStream_t s);
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

cudaError_t launch_transpose_u8(const uint8_t* in, int64_t R, int64_t C, uint8_t* out, cudaStream_t s);

struct P2PSig;
// tcgen05 GEMM: D[M,N] = A[M,K] B[N,K]^T with scales.
//   scale_mode 0: tensor (sa[1], sb[1] float), 1: row (sa[M], sb[N] float), 2: MX (E8M0 blocked)
struct GemmProblem {
  const uint8_t* A; const uint8_t* B;
  int fmt_a, fmt_b;
  int a_mn, b_mn;      // 1: operand stored MN-major ([K,M] / [K,N] row-major)
  const void* sa; const void* sb;
  int scale_mode;
  int64_t M, N, K, lda, ldb;
  void* D; int out_f32; int64_t ldd;
  int bf16_in = 0;     // 1: A and B are BF16 (kind::f16, no scales; rowwise_gw_hp dW)
  uint32_t* out_amax = nullptr;  // optional epilogue amax of |D| (pre-zeroed u32 accumulator)
  // MoE grouped problem (see Prob in gemm_kernels.cu): 1 = M-grouped (fwd, dX), 2 = K-grouped (dW);
  // offs = device int[G+1] group offsets (multiples of 128), G <= GEMM_MAX_GROUPS.
  int grouped = 0;
  int G = 0;
  const int* offs = nullptr;
  // async-TP: per-chunk arrival flags of A's rows (see Prob in gemm_kernels.cu)
  const unsigned long long* chunk_done = nullptr;
  int chunk_rows = 0;
  int mrot = 0;
  unsigned chunk_epoch = 0;
  // fused reduce-scatter of D over row chunks (see Prob in gemm_kernels.cu)
  uint8_t* const* rs_bufs = nullptr;   // device table [P]: every rank's staging buffer
  P2PSig* const* rs_sigs = nullptr;    // device table [P]: every rank's signal block
  unsigned* rs_cnt = nullptr;          // local per-chunk counters (this rank's signal block)
  int rs_rank = 0, rs_chunk_rows = 0, rs_expect = 0;
  unsigned rs_epoch = 0;
};
constexpr int GEMM_MAX_GROUPS = 256;
constexpr int GEMM_MAX_PROBS = 6;   // problems per persistent launch (grouped MoE launches: 2)
cudaError_t launch_gemm(const GemmProblem& p, cudaStream_t st);
// Up to GEMM_MAX_PROBS problems of the same kind (scale mode) on one persistent launch, longest K first.
cudaError_t launch_gemms(const GemmProblem* ps, int n, cudaStream_t st);

}  // namespace fp8t
