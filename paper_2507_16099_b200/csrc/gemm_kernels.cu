// Scaled FP8 GEMM on 5th-generation tensor cores (tcgen05), sm_100a.
//
//   D[m,n] = sum_k dec(A[m,k]) dec(B[n,k]) * epilogue scales
//
// Persistent, warp-specialised, one CTA per SM:
//   warp 0      TMA producer: A/B tiles (SWIZZLE_128B, K-major) into an smem ring; MX: E8M0
//               scale-factor tiles by 1-D bulk copy
//   warp 1      MMA issuer: one thread issues tcgen05.mma (kind::f8f6f4 or
//               kind::mxf8f6f4.block_scale) into a TMEM accumulator; tcgen05.commit frees smem
//               stages and publishes finished accumulators
//   warp 2      TMEM allocator
//   warps 4..7  epilogue: tcgen05.ld 32 lanes x 32 columns -> fp32 -> * (1/sa)(1/sb) ->
//               bf16/fp32 -> global
//
// CG = 2 (default for the plain FP8 kinds): a CTA pair (cluster of 2) computes a 256 x 256
// tile with tcgen05.mma.cta_group::2 (M = 256): each CTA stages its own 128 rows of A and
// half (128 rows) of B, so per-SM operand traffic is 32 KB per 128-deep K block instead of
// 48 KB; the leader CTA issues the MMAs, both CTAs hold 128 accumulator lanes.  A stage holds
// KS = 2 K atoms (256-deep K, 64 KB per CTA, 3 stages): 8 MMAs per full/empty barrier round
// trip, which halves the per-MMA synchronisation overhead of the single-atom ring (measured
// +10-25% on the C2 shapes).
// CG = 1: a single CTA computes 128 x 256 (kept as a reference variant; knob gemm_cta_group = 1).
// Accumulators are double-buffered in TMEM (2 x 256 columns) for the plain FP8 kinds so the
// epilogue of tile i overlaps the mainloop of tile i+1; the MX kind keeps one accumulator
// (256 columns) plus the scale-factor columns (E8M0 tiles loaded by TMA next to the operands,
// tcgen05.cp'd into TMEM per stage; in CTA-pair mode each CTA holds SFA for its own rows and
// SFB for all 256 N rows).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <atomic>
#include <mutex>

#include "kernels.h"
#include "ptx.cuh"

namespace fp8t {

constexpr int BM = 128, BN = 256, BK = 128;   // per-CTA M rows, MMA N, K atom (bytes)
constexpr int SF_CHUNK = 512;                 // E8M0 tile: 128 rows x 4 K-blocks of 32 (one K atom)
constexpr int GROUP_M = 16;                   // grouped raster: 16 M-tiles share the N sweep
constexpr int GMAX = GEMM_MAX_GROUPS;         // MoE grouped GEMM: groups per problem
constexpr int SD = 8;                         // depth of a CTA pair's tile-index ring (see the scheduler)
constexpr int SCHED_SLOTS = 4096;             // launches in flight that may share the counter array

// Dynamic tile scheduler state: [slot][0] = next dynamic tile, [slot][1] = pairs done fetching.  Every
// launch takes its own slot (host-side round robin); the last pair to finish fetching resets both, so a
// slot is zero again when it is reused.  Slots [0, SCHED_SLOTS) serve eager launches, [SCHED_SLOTS,
// 2 SCHED_SLOTS) launches captured into CUDA graphs (a graph keeps its slot for every replay, so eager
// launches never share it).  Module-global device memory: no allocation in any call.
__device__ unsigned g_sched[2 * SCHED_SLOTS][2];

// One GEMM problem of a (possibly two-problem) launch.
struct Prob {
  int M, N, K;
  int tiles_m, tiles_n, num_kb;
  int sf_tiles_k;     // K / 128: 512-byte scale tiles per 128-row block (MX)
  uint32_t idesc;
  const float* sa; const float* sb;
  void* D; int64_t ldd;
  int out_f32, row_scales;
  int d_tma;          // bf16 epilogue writing D by TMA stores through map slot 4 (N = 512 tiles; 256-wide tiles with
                      // knob gemm_epi_tma)
  int a_mn, b_mn;     // operand majors (MN-major: TMA boxes 128 MN x 128 K, K step 4 KB)
  uint32_t* out_amax; // optional: atomicMax of |D| bit patterns (amax of the stored output values)
  int raster;         // tile raster of this problem (see tile_coords / choose_raster)
  // MoE grouped problems (scaled_grouped_mm): offs = device [G+1] row offsets
  //   grouped 1 (M-grouped, fwd / dX): group g owns rows [offs[g], offs[g+1]) of A, D and sa; B is
  //             expert g's block (K-major: rows g*N.., MN-major: K rows g*K..); sb index g*N + col
  //   grouped 2 (K-grouped, dW): group g contracts over rows [offs[g], offs[g+1]) of both MN-major
  //             operands; D rows g*M.., sa index g*M + row, sb index g*N + col; empty group -> 0
  int grouped, G;
  const int* offs;
  // async-TP (fp8_tp_allgather_linear_fwd): rows of A arrive by chunks of chunk_rows pushed by the
  // other ranks; the producer waits for chunk_done[c] >= chunk_epoch before loading chunk c, and
  // M tiles are rotated by mrot so this rank's own chunk is computed first
  const unsigned long long* chunk_done;
  int chunk_rows, mrot;
  unsigned chunk_epoch;
  // fused reduce-scatter (fp8_linear_bwd_rs / fp8_tp_linear_bwd): D's row chunk c (rs_chunk_rows rows)
  // belongs to rank c.  The epilogue stores a tile of chunk c straight into rank c's staging buffer at
  // source slot rs_rank ([P][rs_chunk_rows][N] bf16); each epilogue warp then counts itself on the local
  // chunk counter, and the last of the chunk's rs_expect warps fences at system scope and publishes
  // done[rs_rank] = rs_epoch in rank c's signal block.  Rank c sums its P slots afterwards.
  uint8_t* const* rs_bufs;
  P2PSig* const* rs_sigs;
  unsigned* rs_cnt;
  int rs_rank, rs_chunk_rows, rs_expect;
  unsigned rs_epoch;
};
// A launch processes the tiles of p[0] ([tstart[0] = 0, tstart[1])), then p[1], ... p[np - 1] (up to
// tstart[np] = num_tiles) on one persistent grid: the backward's dX and dW GEMMs share one launch (and a
// shared-input group's members all theirs), so no problem has its own wave-quantisation tail.  Grouped
// (MoE) launches carry at most two problems, whose tile counts are known on the device only.
constexpr int MAXP = GEMM_MAX_PROBS;
struct alignas(64) GemmMaps {
  CUtensorMap m[MAXP][5];   // per problem: A, B, SFA, SFB, D (bf16 output map of the TMA-store epilogue)
};
struct GemmArgs {
  Prob p[MAXP];
  int tstart[MAXP + 1];
  int np, num_tiles;
  int debug;          // bit 0: skip the epilogue's global stores (mainloop-only timing)
  int sf_split;       // MX: scale-factor copies issued by their own warp (see the SF copier)
  int kserp;          // K-serpentine: tiles of odd "waves" (tile / pairs) walk their K stages backwards
  int l2pf;           // L2 prefetch distance of the operand boxes, in stages (0 = off)
  int wsleep;         // knob wait_sleep: bit 1 epilogue waits, bit 2 producer / scheduler waits, bit 3 MMA / SF waits
                      // use the suspend-time-hint try_wait (waiting warps sleep instead of spinning)
  int afill;          // knob gemm_afill: N = 512 tiles issue both halves' MMAs per K step with A kept in the collector
  int l2hint;         // knob gemm_l2hint (A/B): 1 A panels evict_last (the grouped raster reuses them across the
                      // group's N sweep), 2 + B evict_first, 3 A evict_last with B explicitly evict_normal
  int st_ef;          // bf16 outputs stored with an L2 evict-first hint (written back during the GEMM, so the
                      // next memory-bound kernel does not pay for evicting them)
  unsigned* fault;    // process fault word (async-TP watchdog, bad group offsets); may be null
  unsigned long long watchdog_ns;
  unsigned* sched;    // dynamic tile scheduler slot (g_sched[i]); null: static round robin
};

template <bool MX, int CG, int ST, int KS, bool BF = false, bool GRP = false, bool E8 = false, int BNT = 256> struct Layout {
  static constexpr int STAGES = ST;
  // MMA N of a tile.  256 everywhere except the MXFP8 N = 192 variant (K-major operands, CTA pair): two
  // 192-column accumulators + the scale-factor columns fit the 512 TMEM columns, 2 x 256 do not
  // N = 512 (plain FP8 kinds, CTA pair, 1-atom stages): a 256 x 512 tile as two N = 256 MMAs per K step sharing
  // A, i.e. 25 % fewer L2 -> SMEM operand bytes per flop than 256 x 256 (the measured limit at full clock,
  // DESIGN.md §5); the two halves own TMEM columns [0, 256) and [256, 512) of one accumulator and are handed
  // to the epilogue half by half (HALVES).
  static constexpr int BN = BNT;
  static_assert(BN == 256 || (BN == 192 && MX && CG == 2) || (BN == 512 && !MX && !BF && !GRP && CG == 2 && KS == 1),
                "N = 192 tiles: MX CTA-pair kernel only; N = 512: plain FP8 CTA-pair 1-atom kernel only");
  static constexpr int HALVES = BN == 512 ? 2 : 1;
  static constexpr int ACC = (MX && BN == 256) || BN == 512 ? 1 : 2;
  static constexpr int NACC = ACC * HALVES;                   // tfull / tempty barriers
  static constexpr int EPI_WARPS = E8 || ACC == 1 ? 8 : 4;   // see the epilogue
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  // a stage holds KS 128-byte K atoms (16 KB sub-tiles of 128 rows each)
  static constexpr uint32_t A_STAGE = BM * BK * KS;         // 16 KB x KS
  static constexpr uint32_t B_ATOM = ((BN > 256 ? BN : 256) / CG) * BK;   // smem bytes of one B K atom
  static constexpr uint32_t B_STAGE = B_ATOM * KS;  // 32 KB (CG=1, or N = 512) / 16 KB (CG=2) atom slots, x KS
  static constexpr uint32_t B_TX = (BN / CG) * BK * KS;     // bytes actually loaded (N = 192: 12 KB per atom)
  // MX scale factors per stage: SFA = this CTA's 128 rows x KS atoms; SFB = all 256 N rows x KS
  static constexpr uint32_t SFA_STAGE = MX ? KS * SF_CHUNK : 0;
  static constexpr uint32_t SFB_STAGE = MX ? 2 * KS * SF_CHUNK : 0;
  static constexpr uint32_t off_a = 0;
  static constexpr uint32_t off_b = off_a + STAGES * A_STAGE;
  static constexpr uint32_t off_sfa = off_b + STAGES * B_STAGE;
  static constexpr uint32_t off_sfb = off_sfa + STAGES * SFA_STAGE;
  // per epilogue warp: 2 KB bf16 staging for the row-segment stores; N = 512: two 2 KB output chunks (32 rows
  // x 32 bf16 columns, SWIZZLE_64B) written by TMA stores, double-buffered
  static constexpr uint32_t EPI_BYTES = BN == 512 ? 4096 : 2048;
  static constexpr uint32_t off_epi = off_sfb + STAGES * SFB_STAGE;
  static constexpr uint32_t off_bar = off_epi + EPI_WARPS * EPI_BYTES;
  // mbarriers (8 B each), in this order from off_bar; the kernel takes every address from these offsets
  static constexpr uint32_t off_full = off_bar;                                 // [STAGES]
  static constexpr uint32_t off_empty = off_full + 8 * STAGES;                  // [STAGES]
  static constexpr uint32_t off_tfull = off_empty + 8 * STAGES;                 // [NACC]
  static constexpr uint32_t off_tempty = off_tfull + 8 * NACC;                  // [NACC]
  static constexpr uint32_t off_sf_bar = off_tempty + 8 * NACC;                 // [STAGES] (MX only)
  static constexpr uint32_t off_sf_full = off_sf_bar + (MX ? 8 * STAGES : 0);   // [STAGES] (MX only)
  static constexpr uint32_t off_sched_full = off_sf_full + (MX ? 8 * STAGES : 0);   // [SD]
  static constexpr uint32_t off_sched_empty = off_sched_full + 8 * SD;         // [SD]
  static constexpr uint32_t off_tmem = off_sched_empty + 8 * SD;
  // grouped: per problem the group offsets and the prefix of M tiles (ints, 2 x 2 x (GMAX + 1))
  static constexpr uint32_t off_ring = off_tmem + 16;      // [SD] tile indices published by the pair's scheduler
  static constexpr uint32_t off_grp = off_ring + 4 * SD;
  static constexpr uint32_t grp_bytes = GRP ? 16 * (GMAX + 1) : 0;
  static constexpr uint32_t bytes = off_grp + grp_bytes + 1024;  // + alignment slack
  static constexpr uint32_t tmem_cols = 512;
  // MX TMEM columns after the single accumulator, one set per pipeline stage (so the tcgen05.cp of
  // stage s+1 never overwrites columns the MMAs of stage s still read): stage s, SFA atom t at
  // sfa_col + s*SF_COLS + 4t; SFB (row block h, atom t) at sfb_col + s*SF_COLS + 8t + 4h
  static constexpr uint32_t SF_COLS = 12 * KS;
  static constexpr uint32_t sfa_col = ACC * BN, sfb_col = ACC * BN + 4 * KS;
  static_assert(!MX || sfa_col + STAGES * SF_COLS <= 512, "TMEM columns");
  static constexpr uint32_t tx_bytes = CG * (A_STAGE + B_TX);   // operands, counted on the leader
  static constexpr uint32_t sf_tx_bytes = CG * (SFA_STAGE + SFB_STAGE);   // MX scale tiles (sf_full)
};

// Where one output tile of a (possibly grouped) problem lives.
struct TileInfo {
  int pi, mb, nb;
  int m_valid;                     // rows of this problem / group
  int a_row0, a_k0, b_row0, b_k0;  // operand coordinate offsets (grouped problems)
  int num_kb, katoms;              // K stages of the tile, valid 128-deep K atoms
  int64_t d_row0, sa_off, sb_off;  // output row / scale index offsets
};

// Tile raster.  group_m > 0: groups of group_m M-tiles sweep all N tiles (L2 reuse of both
// operands); group_m == 0: row-major (all N tiles of an M tile back to back, so the B operand
// stays L2-resident while A streams through once).
__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int group_m, int& mb, int& nb) {
  if (group_m == 0) {
    mb = t / tiles_n;
    nb = t - mb * tiles_n;
    return;
  }
  const int group = t / (group_m * tiles_n);
  const int first_m = group * group_m;
  const int gsz = min(group_m, tiles_m - first_m);
  const int local = t - group * group_m * tiles_n;
  mb = first_m + local % gsz;
  nb = local / gsz;
}

template <bool MX, int CG, int ST, int KS, bool BF, bool GRP, bool E8, int BNT>
__global__ void __launch_bounds__(Layout<MX, CG, ST, KS, BF, GRP, E8, BNT>::THREADS, 1)
    fp8_gemm_kernel(const __grid_constant__ GemmMaps maps, const __grid_constant__ GemmArgs args) {
  static_assert(KS == 1 || CG == 2, "multi-atom stages need the CTA-pair kernel");
  static_assert(!BF || (CG == 2 && KS == 2 && !MX), "BF16 operands: CTA-pair, 2-atom stages");
  static_assert(!GRP || (!MX && !BF), "grouped problems: plain FP8 kinds");
  using L = Layout<MX, CG, ST, KS, BF, GRP, E8, BNT>;
  constexpr int STAGES = L::STAGES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t full_bar = base + L::off_full;                // [STAGES]  (leader counts both CTAs)
  const uint32_t empty_bar = base + L::off_empty;              // [STAGES]
  const uint32_t tfull_bar = base + L::off_tfull;              // [ACC]
  const uint32_t tempty_bar = base + L::off_tempty;            // [ACC]    (leader counts both CTAs)
  const uint32_t sf_bar = base + L::off_sf_bar;                // [STAGES] MX: stage's scales are in TMEM
  const uint32_t sf_full = base + L::off_sf_full;              // [STAGES] MX: stage's scale tiles in smem
  const uint32_t sched_full = base + L::off_sched_full;        // [SD] ring slot holds the next tile index
  const uint32_t sched_empty = base + L::off_sched_empty;      // [SD] (leader) every consumer has read it
  const uint32_t ring = base + L::off_ring;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + L::off_tmem);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t crank = CG == 2 ? cluster_ctarank() : 0;
  const bool leader = crank == 0;
  const bool sf_split = MX && args.sf_split && !(args.debug & 2);   // (see the SF copier)
  const int cta_slot = CG == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;   // pair / CTA index
  const int cta_stride = CG == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  // grouped problems: smem copies of the offsets and the prefix sums of M tiles per group
  int* goffs = reinterpret_cast<int*>(gbase + L::off_grp);   // [2][GMAX + 1]
  int* gpre = goffs + 2 * (GMAX + 1);                         // [2][GMAX + 1]
  if (GRP && warp == 3 && lane < 2) {
    const Prob& P = args.p[lane];
    int* o = goffs + lane * (GMAX + 1);
    int* pre = gpre + lane * (GMAX + 1);
    if (P.grouped) {
      // group offsets must start at 0, never decrease, be multiples of 128 and end at the
      // grouped extent (rows for grouped 1, the contraction length for grouped 2)
      const int extent = P.grouped == 1 ? P.M : P.K;
      int prev = 0, acc = 0;
      bool ok = __ldg(P.offs) == 0;
      pre[0] = 0;
      for (int g = 0; g <= P.G; ++g) {
        const int v = __ldg(P.offs + g);
        ok = ok && v >= prev && (v & 127) == 0 && v <= extent;
        o[g] = v;
        if (g > 0) {
          acc += (v - prev + BM * CG - 1) / (BM * CG);
          pre[g] = acc;
        }
        prev = v;
      }
      if (!ok || prev != extent) {   // report through the fault word; compute no tile of this problem
        if (blockIdx.x == 0 && args.fault) atomicExch_system(args.fault, fault_pack(FAULT_GROUP_OFFSETS, lane, 0));
        for (int g = 0; g <= P.G; ++g) {
          o[g] = 0;
          pre[g] = 0;
        }
      }
    }
  }
  // problem of a global tile index, its coordinates and offsets
  auto count = [&](const Prob& P, int pi) -> int {
    if (!GRP || P.grouped == 0) return P.tiles_m * P.tiles_n;
    if (P.grouped == 1) return gpre[pi * (GMAX + 1) + P.G] * P.tiles_n;
    return P.G * P.tiles_m * P.tiles_n;
  };
  int t1 = args.tstart[1], num_tiles = args.num_tiles;   // (grouped: known after the setup barrier)
  auto locate = [&](int tile) -> TileInfo {
    TileInfo ti{};
    int pi = 0;
    if (GRP) {
      pi = tile >= t1 ? 1 : 0;
    } else {
      while (pi + 1 < args.np && tile >= args.tstart[pi + 1]) ++pi;
    }
    ti.pi = pi;
    const Prob& P = args.p[pi];
    const int local = tile - (GRP ? (pi ? t1 : 0) : args.tstart[pi]);
    ti.m_valid = P.M;
    ti.num_kb = P.num_kb;
    ti.katoms = 1 << 30;
    if (!GRP || P.grouped == 0) {
      tile_coords(local, P.tiles_m, P.tiles_n, P.raster, ti.mb, ti.nb);
      if (P.mrot) ti.mb = (ti.mb + P.mrot) % P.tiles_m;
      return ti;
    }
    const int* o = goffs + ti.pi * (GMAX + 1);
    int g;
    if (P.grouped == 1) {
      const int* pre = gpre + ti.pi * (GMAX + 1);
      int mi;
      tile_coords(local, pre[P.G], P.tiles_n, P.raster, mi, ti.nb);
      int lo = 0, hi = P.G;   // pre[lo] <= mi < pre[hi]
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (pre[mid] <= mi) lo = mid; else hi = mid;
      }
      g = lo;
      ti.mb = mi - pre[g];
      ti.katoms = (P.K + BK - 1) / BK;   // MN-major B: expert g's contraction rows end at (g+1)*K
      ti.m_valid = o[g + 1] - o[g];
      ti.a_row0 = o[g];
      ti.d_row0 = o[g];
      ti.sa_off = o[g];
      if (P.b_mn) ti.b_k0 = g * P.K; else ti.b_row0 = g * P.N;
      ti.sb_off = (int64_t)g * P.N;
    } else {
      const int per = P.tiles_m * P.tiles_n;
      g = local / per;
      tile_coords(local - g * per, P.tiles_m, P.tiles_n, P.raster, ti.mb, ti.nb);
      ti.a_k0 = o[g];
      ti.b_k0 = o[g];
      ti.katoms = (o[g + 1] - o[g]) / BK;
      ti.num_kb = (ti.katoms + KS - 1) / KS;
      ti.d_row0 = (int64_t)g * P.M;
      ti.sa_off = (int64_t)g * P.M;
      ti.sb_off = (int64_t)g * P.N;
    }
    return ti;
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < args.np; ++i) {
      tma_prefetch_desc(&maps.m[i][0]);
      tma_prefetch_desc(&maps.m[i][1]);
      if (MX) {
        tma_prefetch_desc(&maps.m[i][2]);
        tma_prefetch_desc(&maps.m[i][3]);
      }
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar + 8 * s, CG);
      mbar_init(empty_bar + 8 * s, 1);
    }
    for (int a = 0; a < L::NACC; ++a) {
      mbar_init(tfull_bar + 8 * a, 1);
      mbar_init(tempty_bar + 8 * a, CG * L::EPI_WARPS);   // one arrival per epilogue warp
    }
    if (MX)
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(sf_bar + 8 * s, 1);
        mbar_init(sf_full + 8 * s, CG);
      }
    // consumers of the tile sequence: MMA warp (+ SF copier) and epilogue warps of the leader, plus the
    // peer's producer and epilogue warps; the leader's producer is the scheduler itself
    const uint32_t consumers = 1 + (sf_split ? 1 : 0) + L::EPI_WARPS + (CG == 2 ? 1 + L::EPI_WARPS : 0);
    for (int i = 0; i < SD; ++i) {
      mbar_init(sched_full + 8 * i, 1);
      mbar_init(sched_empty + 8 * i, consumers);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    if (CG == 2) {
      tmem_alloc_cg2(smem_u32(tmem_slot), L::tmem_cols);
      tmem_relinquish_cg2();
    } else {
      tmem_alloc(smem_u32(tmem_slot), L::tmem_cols);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  if (CG == 2) cluster_sync();   // barrier inits and the pair's TMEM allocation visible cluster-wide
  __syncthreads();               // (also the CTA-level barrier racecheck models for the smem slot)
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (GRP) {
    t1 = count(args.p[0], 0);
    num_tiles = t1 + (args.np > 1 ? count(args.p[1], 1) : 0);
  }

  // MX: copy a stage's E8M0 tiles smem -> TMEM (tcgen05.cp; 3 copies of 512 B per K atom, each
  // replicated into the 4 TMEM lane quadrants).  Every stage has its own TMEM columns.
  auto copy_sf = [&](int st, uint32_t tmem_base) {
    const uint32_t ssa = base + L::off_sfa + st * L::SFA_STAGE;
    const uint32_t ssb = base + L::off_sfb + st * L::SFB_STAGE;
#pragma unroll
    for (int t = 0; t < KS; ++t) {
      const uint32_t ca = tmem_base + L::sfa_col + st * L::SF_COLS + 4 * t;
      const uint32_t cb0 = tmem_base + L::sfb_col + st * L::SF_COLS + 8 * t, cb1 = cb0 + 4;
      if (CG == 2) {
        tmem_cp_32x128b_warpx4_cg2(ca, make_sf_desc(ssa + t * SF_CHUNK));
        tmem_cp_32x128b_warpx4_cg2(cb0, make_sf_desc(ssb + t * SF_CHUNK));
        tmem_cp_32x128b_warpx4_cg2(cb1, make_sf_desc(ssb + (KS + t) * SF_CHUNK));
      } else {
        tmem_cp_32x128b_warpx4(ca, make_sf_desc(ssa + t * SF_CHUNK));
        tmem_cp_32x128b_warpx4(cb0, make_sf_desc(ssb + t * SF_CHUNK));
        tmem_cp_32x128b_warpx4(cb1, make_sf_desc(ssb + (KS + t) * SF_CHUNK));
      }
    }
  };
  // sf_split: a separate SF-copier warp issues the copies and commits them to sf_bar[stage]; the MMA
  // warp waits on that barrier.  Measured: when one thread interleaves tcgen05.cp with its MMAs,
  // every cp -> MMA transition costs ~800-1000 cycles (the cost scales with the number of
  // transitions, not of copies), i.e. ~40 % of an 8-MMA stage; tcgen05 ops of different threads
  // are not ordered with each other, so the copier's copies overlap the MMAs in flight.
  // WAR on the stage's TMEM columns: full_bar[stage] of this round implies the producer refilled the
  // slot after empty_bar[stage], i.e. after the MMAs that read the previous round's scales completed.
  // Tile sequence of this CTA (pair).  Persistent CTAs take tiles from a scheduler: the leader's
  // producer publishes each tile index into slot k % SD of both CTAs' rings (sched_full) before loading
  // it; every other role reads the same sequence from its own CTA's ring and releases the slot on the
  // leader (sched_empty).  Index >= num_tiles ends the sequence.  The first tile of a pair is its slot
  // index; later ones come from a global atomic counter (args.sched) in tile order -- the host puts the
  // problem with the longer K first, so long tiles are handed out first and short ones fill the gaps
  // (dynamic, LPT-like) -- or, with args.sched == null, round robin (tile += pairs).
  auto seq_get = [&](int& k) -> int {
    const int slot = k & (SD - 1);
    const uint32_t ph = (uint32_t)(k / SD) & 1u;
    ++k;
    mbar_wait_acq_cluster(sched_full + 8 * slot, ph);
    int t = 0;
    if (lane == 0) t = ld_volatile_shared_s32(ring + 4 * slot);
    t = __shfl_sync(0xffffffffu, t, 0);   // the read has completed before the slot is released
    if (lane == 0) {
      if (CG == 2 && !leader) mbar_arrive_release_cluster(mapa_shared(sched_empty + 8 * slot, 0));
      else mbar_arrive(sched_empty + 8 * slot);
    }
    return t;
  };
  auto seq_put = [&](int& k, int t) {   // leader producer
    const int slot = k & (SD - 1);
    const uint32_t ph = (uint32_t)(k / SD) & 1u;
    ++k;
    mbar_wait_opt(sched_empty + 8 * slot, ph ^ 1u, args.wsleep & 4);
    if (lane == 0) {
      asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(ring + 4 * slot), "r"(t) : "memory");
      if (CG == 2) {
        st_shared_cluster_u32(mapa_shared(ring + 4 * slot, 1), (uint32_t)t);
        mbar_arrive_release_cluster(mapa_shared(sched_full + 8 * slot, 1));
      }
      mbar_arrive(sched_full + 8 * slot);
    }
    __syncwarp();
  };
  // leader producer: the tile after t.  sched_fetch issues lane 0's atomic when tile t's loads start;
  // sched_next consumes its result after them (the atomic's latency hides behind the loads).
  auto sched_fetch = [&]() -> unsigned { return (lane == 0 && args.sched) ? atomicAdd(args.sched, 1u) : 0u; };
  auto sched_next = [&](int t, unsigned fetched) -> int {
    int nt = 0;
    if (lane == 0) {
      if (args.sched) {
        nt = cta_stride + (int)fetched;
        if (nt >= num_tiles && atomicAdd(args.sched + 1, 1u) == (unsigned)cta_stride - 1) {
          atomicExch(args.sched, 0u);   // every pair has done its last fetch: reset the slot
          atomicExch(args.sched + 1, 0u);
        }
      } else {
        nt = t + cta_stride;
      }
    }
    return __shfl_sync(0xffffffffu, nt, 0);
  };

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    const uint64_t polA = l2_policy_evict_last();
    const uint64_t polB = args.l2hint == 2 ? l2_policy_evict_first() : l2_policy_evict_normal();
    int stage = 0;
    uint32_t phase = 0;
    int sk = 0;
    int tile = cta_slot;
    if (leader && args.sched && tile >= num_tiles && lane == 0 &&   // (grouped grids: a pair with no tile)
        atomicAdd(args.sched + 1, 1u) == (unsigned)cta_stride - 1) {
      atomicExch(args.sched, 0u);
      atomicExch(args.sched + 1, 0u);
    }
    for (;;) {
      unsigned fetched = 0;
      if (leader) {
        seq_put(sk, tile);
        if (tile >= num_tiles) break;
        fetched = sched_fetch();
      } else {
        tile = seq_get(sk);
        if (tile >= num_tiles) break;
      }
      const TileInfo ti = locate(tile);
      const int pi = ti.pi, mb = ti.mb, nb = ti.nb;
      const Prob& P = args.p[pi];
      const CUtensorMap* tmA = &maps.m[pi][0];
      const CUtensorMap* tmB = &maps.m[pi][1];
      const CUtensorMap* tmSFA = &maps.m[pi][2];
      const CUtensorMap* tmSFB = &maps.m[pi][3];
      const int a_mn = P.a_mn, b_mn = P.b_mn;
      const int m0 = mb * BM * CG + (int)crank * BM;
      const int n0 = nb * L::BN + (int)crank * (L::BN / CG);
      // debug bit 4: skip the MX scale-factor loads (timing experiments only; results invalid)
      // debug bit 256 (timing experiment, results invalid): no operand loads, the stage completes on arrivals
      const uint32_t tx = (args.debug & 256) ? 0u : L::tx_bytes;
      const uint32_t sf_tx = (args.debug & 4) ? 0u : L::sf_tx_bytes;
      const int KT = P.sf_tiles_k;
      const int num_kb = ti.num_kb;
      // K-serpentine (not for grouped problems): consecutive waves of tiles share operand panels (the
      // grouped raster keeps M blocks across waves), so a wave that walks K in the opposite direction
      // starts on the K slices the previous wave read last -- still in L2 -- instead of re-reading the
      // panels from DRAM.  The direction is a function of the tile index only (deterministic results).
      const bool krev = !GRP && args.kserp && ((tile / cta_stride) & 1);
      if (P.chunk_done) {   // async-TP: wait until the rank that owns these A rows has pushed them
        if (lane == 0) {
          const unsigned long long* f = P.chunk_done + (m0 + ti.a_row0) / P.chunk_rows;
          uint64_t t0;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
          while (ld_acquire_sys_u64(f) < P.chunk_epoch) {
            __nanosleep(64);
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (args.watchdog_ns && args.fault && t - t0 > args.watchdog_ns) {   // give up: report, load anyway
              atomicExch_system(args.fault, fault_pack(FAULT_TP_CHUNK_WAIT, (m0 + ti.a_row0) / P.chunk_rows,
                                                       P.chunk_epoch));
              __threadfence_system();
              break;
            }
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");   // generic-proxy acquire -> TMA reads
        }
        __syncwarp();
      }
      for (int kbi = 0; kbi < num_kb; ++kbi) {
        const int kb = krev ? num_kb - 1 - kbi : kbi;
        // knob gemm_l2pf = d > 0: before waiting for a free stage, ask L2 for the operand boxes d stages
        // ahead, so a stage's TMA load finds its data in L2 (the operand fetch is latency-bound, §5)
        if (!GRP && !BF && args.l2pf && lane == 0 && kbi + args.l2pf < num_kb && !(args.debug & 256)) {
          const int kp = kbi + args.l2pf, kbp = krev ? num_kb - 1 - kp : kp;
#pragma unroll
          for (int j = 0; j < KS; ++j) {
            const int k0 = (kbp * KS + j) * BK;
            tma_prefetch_l2_2d(tmA, a_mn ? m0 : k0, a_mn ? k0 : m0);
            tma_prefetch_l2_2d(tmB, b_mn ? n0 : k0, b_mn ? k0 : n0);
            if (b_mn && L::BN / CG > 128) tma_prefetch_l2_2d(tmB, n0 + 128, k0);
          }
        }
        mbar_wait_opt(empty_bar + 8 * stage, phase ^ 1, args.wsleep & 4);
        if (lane == 0) {
          // MX: E8M0 tiles first, on their own barrier: they land long before the operands, so the SF
          // copier has them in TMEM by the time the MMA warp sees full_bar
          const uint32_t sfb = sf_full + 8 * stage;
          if (MX) {
            if (CG == 2) {
              if (leader) mbar_arrive_expect_tx(sfb, sf_tx);
              else mbar_arrive_cluster(mapa_shared(sfb, 0));
            } else {
              mbar_arrive_expect_tx(sfb, sf_tx);
            }
          }
          if (MX && !(args.debug & 4)) {
            // E8M0 tiles: SF tensor = [row_block * KT + k_atom][512 B]; boxes of KS consecutive atoms
            const int kt0 = kb * KS;
            const uint32_t dsa = base + L::off_sfa + stage * L::SFA_STAGE;
            const uint32_t dsb = base + L::off_sfb + stage * L::SFB_STAGE;
            const int rba = mb * CG + (int)crank;   // this CTA's 128-row block of A
            if (CG == 2) {
              tma_load_2d_2sm(dsa, tmSFA, 0, rba * KT + kt0, sfb);
              // the tile's N rows span 128-row scale blocks c0, c0 + 1 (N = 192: odd tiles start half-way
              // into block c0; the MMA then reads SFB two TMEM columns further)
              const int c0 = L::BN == 256 ? 2 * nb : (3 * nb) >> 1;
              tma_load_2d_2sm(dsb, tmSFB, 0, c0 * KT + kt0, sfb);
              tma_load_2d_2sm(dsb + KS * SF_CHUNK, tmSFB, 0, (c0 + 1) * KT + kt0, sfb);
            } else {
              tma_load_2d(dsa, tmSFA, 0, rba * KT + kt0, sfb, 0);
              tma_load_2d(dsb, tmSFB, 0, (2 * nb) * KT + kt0, sfb, 0);
              tma_load_2d(dsb + KS * SF_CHUNK, tmSFB, 0, (2 * nb + 1) * KT + kt0, sfb, 0);
            }
          }
          const uint32_t fb = full_bar + 8 * stage;
          const uint32_t sa_dst = base + L::off_a + stage * L::A_STAGE;
          const uint32_t sb_dst = base + L::off_b + stage * L::B_STAGE;
          if (CG == 2) {
            if (leader) mbar_arrive_expect_tx(fb, tx);
            else mbar_arrive_cluster(mapa_shared(fb, 0));
          } else {
            mbar_arrive_expect_tx(fb, tx);
          }
          // K-major boxes: (k, row); MN-major boxes: (mn, k), one per 128-wide MN atom.
          // K atom j of this stage starts at k0 = (kb*KS + j)*BK; atoms are 16 KB apart in smem.
#pragma unroll
          for (int j = 0; j < ((args.debug & 256) ? 0 : KS); ++j) {
            // FP8: atom j = K bytes [(kb*KS + j)*128, +128) (MN-major: 128 K rows of 128 MN bytes).
            // BF16: K-major atom j = K elements [(kb*KS + j)*64, +64); MN-major: the stage covers
            // 128 K rows and atom j is MN elements [mn0 + 64j, +64).
            const int k0 = BF ? (kb * KS + j) * 64 : (kb * KS + j) * BK;
            const int kmn = BF ? kb * 128 : k0;          // K row of an MN-major box
            const int am = BF ? m0 + 64 * j : m0, bn = BF ? n0 + 64 * j : n0;
            const uint32_t da = sa_dst + j * 16384, db = sb_dst + j * L::B_ATOM;
            if (CG == 2) {
              if (GRP) {   // grouped problems: per-group row / K offsets into the shared maps
                tma_load_2d_2sm(da, tmA, a_mn ? am + ti.a_row0 : k0 + ti.a_k0,
                                a_mn ? kmn + ti.a_k0 : m0 + ti.a_row0, fb);
                tma_load_2d_2sm(db, tmB, b_mn ? bn + ti.b_row0 : k0 + ti.b_k0,
                                b_mn ? kmn + ti.b_k0 : n0 + ti.b_row0, fb);
              } else if (args.l2hint) {
                tma_load_2d_2sm_hint(da, tmA, a_mn ? am : k0, a_mn ? kmn : m0, fb, polA);
                tma_load_2d_2sm_hint(db, tmB, b_mn ? bn : k0, b_mn ? kmn : n0, fb, polB);
                if (b_mn && L::BN / CG > 128) tma_load_2d_2sm_hint(db + 16384, tmB, bn + 128, kmn, fb, polB);
              } else {
                tma_load_2d_2sm(da, tmA, a_mn ? am : k0, a_mn ? kmn : m0, fb);
                tma_load_2d_2sm(db, tmB, b_mn ? bn : k0, b_mn ? kmn : n0, fb);
                // N = 512: this CTA's 256 B rows are one 256-row K-major box or two 128-wide MN-major boxes
                if (b_mn && L::BN / CG > 128) tma_load_2d_2sm(db + 16384, tmB, bn + 128, kmn, fb);
              }
            } else {
              tma_load_2d(da, tmA, a_mn ? m0 : k0, a_mn ? k0 : m0, fb, 0);
              if (b_mn) {
                tma_load_2d(db, tmB, n0, k0, fb, 0);
                tma_load_2d(db + 16384, tmB, n0 + 128, k0, fb, 0);
              } else {
                tma_load_2d(db, tmB, k0, n0, fb, 0);
              }
            }
          }
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (leader) tile = sched_next(tile, fetched);
    }
  } else if (warp == 1 && leader) {
    // ---------------- MMA issuer (leader CTA) ----------------
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    // The next tile's index and coordinates are fetched two stages before the current tile's last
    // MMAs are issued, so that bookkeeping overlaps MMAs already queued in the tensor pipe.
    int sk = 0;
    int tile = seq_get(sk);
    TileInfo ti{};
    if (tile < num_tiles) ti = locate(tile);
    while (tile < num_tiles) {
      const Prob& P = args.p[ti.pi];
      const int a_mn = P.a_mn, b_mn = P.b_mn, num_kb = ti.num_kb;
      const uint32_t idesc = P.idesc;
      int next = 0;
      bool have_next = false;
      TileInfo nti{};
      auto fetch_next = [&]() {
        next = seq_get(sk);
        if (next < num_tiles) nti = locate(next);
        have_next = true;
      };
      // N = 512: the tile's two N = 256 halves are handed over separately -- half 1's columns are awaited
      // only after half 0's MMAs of the first stage are queued, and half 0 is published to the epilogue
      // before half 1's MMAs of the last stage -- so each hand-over overlaps the other half's MMAs
      mbar_wait_opt(tempty_bar + 8 * acc * L::HALVES, acc_phase ^ 1, args.wsleep & 8);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * L::BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        if (!have_next && kb + 2 >= num_kb) fetch_next();
        mbar_wait_opt(full_bar + 8 * stage, phase, args.wsleep & 8);
        if (sf_split) mbar_wait_opt(sf_bar + 8 * stage, phase, args.wsleep & 8);
        else if (MX) mbar_wait_opt(sf_full + 8 * stage, phase, args.wsleep & 8);
        tc_fence_after();
        if (lane == 0) {
          // debug bits 16/32/64 (timing experiments only; results invalid): duplicate every stage's
          // copies / copy on every 2nd / every 4th stage only
          if (MX && !sf_split && !(args.debug & 2) && !((args.debug & 32) && (kb & 1)) && !((args.debug & 64) && (kb & 3))) {
            copy_sf(stage, tmem_base);
            if (args.debug & 16) copy_sf(stage, tmem_base);
          }
          const uint32_t sa_src = base + L::off_a + stage * L::A_STAGE;
          const uint32_t sb_src = base + L::off_b + stage * L::B_STAGE;
          const uint64_t adesc = a_mn ? make_sw128_mnmajor_desc(sa_src) : make_sw128_kmajor_desc(sa_src);
          const uint64_t bdesc = b_mn ? make_sw128_mnmajor_desc(sb_src) : make_sw128_kmajor_desc(sb_src);
          // per K=32 step: K-major advances 32 B inside the 128-B swizzle row and jumps 16 KB
          // (1024 in 16-B units) to the next K atom every 4 steps; MN-major advances 32 K-rows
          // = 4 KB per step (atoms are contiguous)
          // (BF16 MN-major: 16 K rows = 2 KB per step inside one MN atom; atoms are LBO = 16 KB apart)
          auto koff = [](int mn, int k) -> uint64_t {
            return mn ? (uint64_t)((BF ? 128 : 256) * k) : (uint64_t)(1024 * (k >> 2) + 2 * (k & 3));
          };
          if constexpr (L::HALVES == 2) {
            if (args.afill) {
              // knob gemm_afill: per K step both halves' MMAs back to back, A held in the collector buffer
              // (read from smem once for the two MMAs); half 1 is awaited after half 0's first MMA is queued
              // and half 0 is published before half 1's last MMA, as below
#pragma unroll
              for (int k = 0; k < BK / 32; ++k) {
                const uint64_t ad = adesc + koff(a_mn, k);
                mma_f8f6f4_cg2_afill(d_tmem, ad, bdesc + koff(b_mn, k), idesc, (kb | k) != 0);
                if (k == 0 && kb == 0) {
                  mbar_wait(tempty_bar + 8, acc_phase ^ 1);
                  tc_fence_after();
                }
                if (k == BK / 32 - 1 && kb == num_kb - 1) mma_commit_cg2_mc(tfull_bar, 0x3);
                mma_f8f6f4_cg2_alastuse(d_tmem + 256, ad, bdesc + (uint64_t)(16384 >> 4) + koff(b_mn, k), idesc,
                                        (kb | k) != 0);
              }
            } else
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (h == 1 && kb == 0) {
                mbar_wait(tempty_bar + 8, acc_phase ^ 1);
                tc_fence_after();
              }
              // half h: this CTA's B rows [128 h, 128 h + 128) (16 KB further in the stage), TMEM columns 256 h..
              const uint64_t bdh = bdesc + (uint64_t)((16384 * h) >> 4);
#pragma unroll
              for (int k = 0; k < BK / 32; ++k)
                mma_f8f6f4_cg2(d_tmem + 256 * h, adesc + koff(a_mn, k), bdh + koff(b_mn, k), idesc, (kb | k) != 0);
              if (h == 0 && kb == num_kb - 1) mma_commit_cg2_mc(tfull_bar, 0x3);
            }
          } else
#pragma unroll
          for (int k = 0; k < KS * BK / 32; ++k) {
            if (GRP && kb * KS + (k >> 2) >= ti.katoms) break;   // K-grouped: the group's last atom ends here
            const uint64_t ad = adesc + koff(a_mn, k), bd = bdesc + koff(b_mn, k);
            const uint32_t acc_flag = (kb | k) != 0;
            if (MX) {
              const uint32_t t = (uint32_t)k >> 2;
              const uint32_t id = idesc_with_sf_id(idesc, k & 3, k & 3);
              const uint32_t sfa = tmem_base + L::sfa_col + stage * L::SF_COLS + 4 * t;
              const uint32_t sfb = tmem_base + L::sfb_col + stage * L::SF_COLS + 8 * t + (L::BN == 192 ? 2 * (ti.nb & 1) : 0);
              if (CG == 2) mma_mxf8f6f4_cg2(d_tmem, ad, bd, id, acc_flag, sfa, sfb);
              else mma_mxf8f6f4(d_tmem, ad, bd, id, acc_flag, sfa, sfb);
            } else if (BF) {
              mma_f16_cg2(d_tmem, ad, bd, idesc, acc_flag);
            } else if (CG == 2) {
              mma_f8f6f4_cg2(d_tmem, ad, bd, idesc, acc_flag);
            } else {
              mma_f8f6f4(d_tmem, ad, bd, idesc, acc_flag);
            }
          }
          if (CG == 2) {
            mma_commit_cg2_mc(empty_bar + 8 * stage, 0x3);
            if (kb == num_kb - 1) mma_commit_cg2_mc(tfull_bar + 8 * (acc * L::HALVES + L::HALVES - 1), 0x3);
          } else {
            mma_commit(empty_bar + 8 * stage);
            if (kb == num_kb - 1) mma_commit(tfull_bar + 8 * acc);
          }
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (GRP && num_kb == 0) {   // empty K group: no MMAs; publish the (unused) accumulator at once
        if (lane == 0) {
          if (CG == 2) mma_commit_cg2_mc(tfull_bar + 8 * acc, 0x3);
          else mma_commit(tfull_bar + 8 * acc);
        }
        __syncwarp();
      }
      if (!have_next) fetch_next();
      if (++acc == L::ACC) { acc = 0; acc_phase ^= 1; }
      tile = next;
      ti = nti;
    }
  } else if (MX && warp == 3 && leader && sf_split) {
    // ---------------- SF copier (leader CTA, MX) ----------------
    // (batching the copies of two stages behind one wait was measured slower: the MMAs of the
    // batch's first stage then wait for its second stage to land)
    int stage = 0;
    uint32_t phase = 0;
    for (int sk = 0;;) {
      const int tile = seq_get(sk);
      if (tile >= num_tiles) break;
      const int num_kb = locate(tile).num_kb;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait_opt(sf_full + 8 * stage, phase, args.wsleep & 8);
        tc_fence_after();
        if (lane == 0) {
          copy_sf(stage, tmem_base);
          if (CG == 2) mma_commit_cg2_mc(sf_bar + 8 * stage, 0x1);
          else mma_commit(sf_bar + 8 * stage);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs, own 128 accumulator lanes) ----------------
    // EPIW = 4: one warp per TMEM lane quadrant, 8 chunks of 32 columns, TMEM released after the
    //           tile (the other accumulator buffer keeps the MMAs busy meanwhile).
    // EPIW = 8 (single-accumulator MX kernel; short-K launches): two warps per quadrant, 128 columns
    //           each, loaded into registers and TMEM released BEFORE scaling/storing, so the next
    //           tile's MMAs start after the TMEM drain instead of after the whole epilogue, and twice
    //           the warps share the stores.  Measured (tools/mx_probe.py, flop/clk/SM): K = 1024
    //           (Llama-3-8B wk/wv dX) 7.5k -> 8.6k with 8 warps; K >= 2048 shapes 1-7 % better with 4.
    constexpr int EPIW = L::EPI_WARPS;
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int half = EPIW == 8 ? ((warp - 4) >> 2) : 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint32_t tempty_leader = CG == 2 ? mapa_shared(tempty_bar, 0) : tempty_bar;
    uint8_t* epi = gbase + L::off_epi + (warp - 4) * L::EPI_BYTES;   // this warp's bf16 staging slot
    const uint32_t epi_s = base + L::off_epi + (warp - 4) * L::EPI_BYTES;
    const bool st_ef = args.st_ef != 0;
    const uint64_t st_pol = l2_policy_evict_first();
    for (int sk = 0;;) {
      const int tile = seq_get(sk);
      if (tile >= num_tiles) break;
      const TileInfo ti = locate(tile);
      const int mb = ti.mb, nb = ti.nb;
      const Prob& P = args.p[ti.pi];
      const int N = P.N, row_scales = P.row_scales, out_f32 = P.out_f32;
      const float* sb = P.sb + ti.sb_off;
      const int row = mb * BM * CG + (int)crank * BM + q * 32 + (int)lane;   // row within the problem / group
      const bool rvalid = row < ti.m_valid;
      const bool kzero = GRP && ti.katoms == 0;   // empty K group: D = 0
      float rs = 1.f;
      if (!row_scales && P.sa) rs = __frcp_rn(P.sa[0]) * __frcp_rn(P.sb[0]);
      if (row_scales && rvalid) rs = __frcp_rn(P.sa[ti.sa_off + row]);
      uint8_t* Dbase = static_cast<uint8_t*>(P.D) + ti.d_row0 * P.ldd * (out_f32 ? 4 : 2);
      const int rs_chunk = P.rs_bufs ? (mb * BM * CG) / P.rs_chunk_rows : 0;
      if (P.rs_bufs)   // the tile's rows go to rank rs_chunk's staging slot rs_rank
        Dbase = P.rs_bufs[rs_chunk] + (int64_t)(P.rs_rank - rs_chunk) * P.rs_chunk_rows * P.ldd * (out_f32 ? 4 : 2);
      uint32_t dmax = 0;   // |D| max over this thread's stored values (fp32 bit patterns)

      // scale + convert + store 32 columns [col0, col0 + 32) of this thread's row
      auto process = [&](const uint32_t (&r)[32], int col0) {
        if (col0 >= N || (args.debug & 1)) return;   // warp-uniform
        const int nvalid = min(32, N - col0);  // 16 or 32 (N % 16 == 0)
        uint32_t pk[16];
        bool packed = false;
        if constexpr (MX) {   // block scales are applied inside the MMA (rs = 1, exact): convert straight from TMEM
          if (!out_f32) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
              pk[j] = *reinterpret_cast<uint32_t*>(&h);
            }
            packed = true;
          }
        }
        if (!packed) {
        float v[32];
        if (kzero) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.f;
        } else if (row_scales) {
          // lane j computes 1/sb for column col0 + j once and parks it in the warp's (free) staging buffer; every
          // lane reads the 32 values back as 8 broadcast 16-byte loads (instead of 32 shuffles).  Two columns per
          // __fmul2_rn (IEEE RN per lane: the same roundings, in the same order, as two __fmul_rn)
          reinterpret_cast<float*>(epi)[lane] = __frcp_rn(sb[min(col0 + (int)lane, N - 1)]);
          __syncwarp();
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4) {
            const float4 c4 = reinterpret_cast<const float4*>(epi)[q4];
            const int j = 4 * q4;
            const float2 a0 = __fmul2_rn(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), make_float2(rs, rs));
            const float2 a1 = __fmul2_rn(make_float2(__uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])), make_float2(rs, rs));
            const float2 p0 = __fmul2_rn(a0, make_float2(c4.x, c4.y));
            const float2 p1 = __fmul2_rn(a1, make_float2(c4.z, c4.w));
            v[j] = p0.x; v[j + 1] = p0.y; v[j + 2] = p1.x; v[j + 3] = p1.y;
          }
          __syncwarp();   // every lane has read the scales before the staging writes below reuse the buffer
        } else {
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float2 p2 = __fmul2_rn(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), make_float2(rs, rs));
            v[j] = p2.x;
            v[j + 1] = p2.y;
          }
        }
        if (out_f32) {
          if (!rvalid) return;
          float* dst = reinterpret_cast<float*>(Dbase) + (int64_t)row * P.ldd + col0;
          if (P.out_amax) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < nvalid) dmax = max(dmax, __float_as_uint(v[j]) & 0x7FFFFFFFu);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (4 * j < nvalid)
              reinterpret_cast<float4*>(dst)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          return;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
          pk[j] = *reinterpret_cast<uint32_t*>(&h);
        }
        }
        if (P.out_amax && rvalid) {   // amax of the bf16-rounded outputs (what a consumer reads)
          uint32_t m2 = 0;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (2 * j < nvalid) m2 = __vmaxu2(m2, pk[j] & 0x7FFF7FFFu);
          dmax = max(dmax, max(m2 & 0xFFFFu, m2 >> 16) << 16);
        }
        // Stage this warp's 32 rows x 64 B through smem so each global store instruction writes
        // whole 64-B row segments (8 rows per instruction) instead of 32 scattered 16-B pieces.
        // 16-B unit j of row l sits at l*64 + ((j ^ ((l >> 1) & 3)) * 16): conflict-free both ways.
#pragma unroll
        for (int j = 0; j < 4; ++j)
          *reinterpret_cast<uint4*>(epi + lane * 64 + ((j ^ ((lane >> 1) & 3)) * 16)) =
              make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        __syncwarp();
        // row 8 i + (lane >> 2) of the warp's 32: one 64-bit base per chunk, 8 rows further per store
        const int jq = lane & 3;
        const int grow0 = row - (int)lane + ((int)lane >> 2);
        __nv_bfloat16* dq = reinterpret_cast<__nv_bfloat16*>(Dbase) + (int64_t)grow0 * P.ldd + col0 + 8 * jq;
        const int64_t dstep = 8 * P.ldd;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int rr = 8 * i + ((int)lane >> 2);
          const uint4 val = *reinterpret_cast<const uint4*>(epi + rr * 64 + ((jq ^ ((rr >> 1) & 3)) * 16));
          if (grow0 + 8 * i < ti.m_valid && 8 * jq < nvalid) {
            uint4* dp = reinterpret_cast<uint4*>(dq + i * dstep);
            if (st_ef) st_global_v4_hint(dp, val, st_pol);
            else *dp = val;
          }
        }
        __syncwarp();
      };

      // 256-wide tiles with knob gemm_epi_tma: a 32-column chunk of this warp's 32 rows is scaled into the warp's
      // single 2 KB smem buffer (SWIZZLE_64B rows of 64 B) and leaves by one TMA store; the buffer is reused once
      // the previous store has read it
      const int row_base_w = mb * BM * CG + (int)crank * BM + q * 32;
      auto tma_chunk = [&](const uint32_t (&r)[32], int colc) {
        if (colc >= N || (args.debug & 1)) return;   // warp-uniform
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // buffer free
        __syncwarp();
        const float rcol = row_scales ? __frcp_rn(sb[min(colc + (int)lane, N - 1)]) : 1.f;
        const int nvalid = min(32, N - colc);
        uint32_t m2 = 0;
        uint8_t* buf = epi + lane * 64;
        // 8 columns at a time: scale (two per __fmul2_rn), convert, one 16-byte smem store -- few live registers
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint32_t w[4];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int jc = 8 * u + 2 * jj;
            float2 p2 = __fmul2_rn(make_float2(__uint_as_float(r[jc]), __uint_as_float(r[jc + 1])), make_float2(rs, rs));
            if (row_scales)
              p2 = __fmul2_rn(p2, make_float2(__shfl_sync(0xffffffffu, rcol, jc), __shfl_sync(0xffffffffu, rcol, jc + 1)));
            __nv_bfloat162 hv = __floats2bfloat162_rn(p2.x, p2.y);
            w[jj] = *reinterpret_cast<uint32_t*>(&hv);
            if (P.out_amax && jc < nvalid) m2 = __vmaxu2(m2, w[jj] & 0x7FFF7FFFu);
          }
          *reinterpret_cast<uint4*>(buf + ((u ^ (int)((lane >> 1) & 3)) * 16)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        if (P.out_amax && rvalid) dmax = max(dmax, max(m2 & 0xFFFFu, m2 >> 16) << 16);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          const CUtensorMap* dm = &maps.m[ti.pi][4];
          if (st_ef) tma_store_2d_hint(dm, epi_s, colc, (int)(ti.d_row0 + row_base_w), st_pol);
          else tma_store_2d(dm, epi_s, colc, (int)(ti.d_row0 + row_base_w));
          bulk_commit_group();
        }
      };

      // this warp's accumulator barrier: per buffer, or per half of the N = 512 accumulator
      // (N = 512: the halves are awaited one by one below)
      if (L::HALVES == 1) {
        mbar_wait_opt(tfull_bar + 8 * acc, acc_phase, args.wsleep & 2);
        tc_fence_after();
      }
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * L::BN;
      if (args.debug & 8) {   // timing experiment (results invalid): release the accumulator untouched
        for (int h = 0; h < L::HALVES; ++h) {
          const int ab = L::HALVES == 2 ? h : acc;
          if (L::HALVES == 2) mbar_wait_opt(tfull_bar + 8 * ab, acc_phase, args.wsleep & 2);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (CG == 2) mbar_arrive_cluster(tempty_leader + 8 * ab);
            else mbar_arrive(tempty_bar + 8 * ab);
          }
        }
      } else if (L::HALVES == 2) {
        // N = 512: the accumulator's halves h = 0, 1 (TMEM columns 256 h.., the MMA of B rows 128 h.. of each
        // CTA) are drained in turn by all 8 warps: warp quarter `half` takes columns [128 half, +128) of the
        // half, i.e. tile columns 128 h.. (half 0, CTA 0's B rows) or 256 + 128 h.. (half 1, CTA 1's rows).
        // bf16 outputs are scaled into one of this warp's two 2 KB smem chunks and written by a TMA store each,
        // so the warp never waits on global writes (which compete with the operand loads for L2) before it
        // releases TMEM; a chunk buffer is reused once its previous store has been read out of smem.
        const CUtensorMap* dmap = &maps.m[ti.pi][4];
        const bool tma_out = P.d_tma;
        const int row_base = mb * BM * CG + (int)crank * BM + q * 32;
        for (int h = 0; h < 2; ++h) {
          mbar_wait_opt(tfull_bar + 8 * h, acc_phase, args.wsleep & 2);
          tc_fence_after();
          const uint32_t tb = tbase + 256 * h + 128 * half;
          const int col0 = nb * L::BN + (half == 0 ? 128 * h : 256 + 128 * h);
          // scale + convert 32 columns into chunk buffer c & 1 (SWIZZLE_64B rows of 64 B) and store it by TMA
          auto stage = [&](const uint32_t (&r)[32], int c) {
            if (!tma_out) {
              process(r, col0 + 32 * c);
              return;
            }
            float v[32];
            if (row_scales) {   // column scales through the chunk buffer (broadcast loads), as in process()
              if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");   // buffer c & 1 free
              __syncwarp();
              float* rcb = reinterpret_cast<float*>(epi + (c & 1) * 2048);
              rcb[lane] = __frcp_rn(sb[col0 + 32 * c + (int)lane]);
              __syncwarp();
#pragma unroll
              for (int q4 = 0; q4 < 8; ++q4) {
                const float4 c4 = reinterpret_cast<const float4*>(rcb)[q4];
                const int j = 4 * q4;
                const float2 a0 = __fmul2_rn(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), make_float2(rs, rs));
                const float2 a1 = __fmul2_rn(make_float2(__uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])), make_float2(rs, rs));
                const float2 p0 = __fmul2_rn(a0, make_float2(c4.x, c4.y));
                const float2 p1 = __fmul2_rn(a1, make_float2(c4.z, c4.w));
                v[j] = p0.x; v[j + 1] = p0.y; v[j + 2] = p1.x; v[j + 3] = p1.y;
              }
              __syncwarp();
            } else {
#pragma unroll
              for (int j = 0; j < 32; j += 2) {
                const float2 p2 = __fmul2_rn(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), make_float2(rs, rs));
                v[j] = p2.x;
                v[j + 1] = p2.y;
              }
            }
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              __nv_bfloat162 hv = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
              pk[j] = *reinterpret_cast<uint32_t*>(&hv);
            }
            if (P.out_amax && rvalid) {
              uint32_t m2 = 0;
#pragma unroll
              for (int j = 0; j < 16; ++j) m2 = __vmaxu2(m2, pk[j] & 0x7FFF7FFFu);
              dmax = max(dmax, max(m2 & 0xFFFFu, m2 >> 16) << 16);
            }
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");   // buffer c & 1 free
            __syncwarp();
            uint8_t* buf = epi + (c & 1) * 2048 + lane * 64;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              *reinterpret_cast<uint4*>(buf + ((u ^ (int)((lane >> 1) & 3)) * 16)) =
                  make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (st_ef) tma_store_2d_hint(dmap, epi_s + (c & 1) * 2048, col0 + 32 * c, (int)(ti.d_row0 + row_base), st_pol);
              else tma_store_2d(dmap, epi_s + (c & 1) * 2048, col0 + 32 * c, (int)(ti.d_row0 + row_base));
              bulk_commit_group();
            }
          };
          uint32_t ra[32], rb[32];
          tmem_ld_32x32b_x32(tb, ra);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 4; c += 2) {
            tmem_ld_32x32b_x32(tb + 32 * (c + 1), rb);
            stage(ra, c);
            tmem_wait_ld();
            if (c + 2 < 4) tmem_ld_32x32b_x32(tb + 32 * (c + 2), ra);
            stage(rb, c + 1);
            tmem_wait_ld();
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (CG == 2) mbar_arrive_cluster(tempty_leader + 8 * h);
            else mbar_arrive(tempty_bar + 8 * h);
          }
        }
      } else if (EPIW == 8) {
        constexpr int HC = L::BN / 64;   // 32-column chunks per half
        uint32_t r[HC][32];
#pragma unroll
        for (int c = 0; c < HC; ++c) tmem_ld_32x32b_x32(tbase + half * (L::BN / 2) + c * 32, r[c]);
        tmem_wait_ld();
        tc_fence_before();   // TMEM drained: release it to the MMA warp before the stores
        __syncwarp();
        if (lane == 0) {
          if (CG == 2) mbar_arrive_cluster(tempty_leader + 8 * acc);
          else mbar_arrive(tempty_bar + 8 * acc);
        }
        if (L::HALVES == 1 && P.d_tma) {
#pragma unroll
          for (int c = 0; c < HC; ++c) tma_chunk(r[c], nb * L::BN + half * (L::BN / 2) + c * 32);
        } else {
#pragma unroll
          for (int c = 0; c < HC; ++c) process(r[c], nb * L::BN + half * (L::BN / 2) + c * 32);
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < L::BN / 32; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tbase + c * 32, r);
          tmem_wait_ld();
          if (L::HALVES == 1 && P.d_tma) tma_chunk(r, nb * L::BN + c * 32);
          else process(r, nb * L::BN + c * 32);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (CG == 2) mbar_arrive_cluster(tempty_leader + 8 * acc);
          else mbar_arrive(tempty_bar + 8 * acc);
        }
      }
      if (P.out_amax) {   // (P is uniform across the CTA; every lane reaches this point)
        dmax = __reduce_max_sync(0xffffffffu, dmax);
        if (lane == 0 && dmax) atomicMax(P.out_amax, dmax);
      }
      if (P.rs_bufs) {    // fused reduce-scatter: this warp's rows of the tile are stored
        __syncwarp();
        if (lane == 0) {
          __threadfence_system();
          if (atomicAdd(P.rs_cnt + rs_chunk, 1u) == (unsigned)P.rs_expect - 1) {   // chunk complete
            P.rs_cnt[rs_chunk] = 0;
            __threadfence_system();
            st_release_sys_u64(&P.rs_sigs[rs_chunk]->done[P.rs_rank], P.rs_epoch);
          }
        }
      }
      if (++acc == L::ACC) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) bulk_wait_all0();   // this warp's TMA stores (if any) are complete
  }

  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if (CG == 2) tmem_dealloc_cg2(tmem_base, L::tmem_cols);
    else tmem_dealloc(tmem_base, L::tmem_cols);
  }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
// The tensor-map encode is a driver-API call and fails with CUDA_ERROR_INVALID_CONTEXT on a thread that
// has no current context yet -- e.g. PyTorch's autograd worker when an MX backward is its first CUDA work
// (the runtime binds the device's primary context to a thread only at its first context-using call).
// cudaSetDevice on the thread's current device binds it (CUDA 12: it initialises and makes current the
// primary context; unlike cudaFree it is not a memory operation, so it is harmless inside a stream capture).
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  thread_local bool bound = false;
  if (!bound) {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaSetDevice(dev);
    bound = true;
  }
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D u8 tensor map with SWIZZLE_128B.  K-major operand [rows, K]: dims {K, rows}, box {BK, box_rows}.
// MN-major operand stored [K, MN]: dims {MN, K}, box {128, BK}.
// (BF16 operands: elements of 2 bytes, boxes of 64 elements = 128 bytes along the contiguous dim;
//  ld is in elements and converted to bytes here)
static bool make_operand_map(CUtensorMap* m, const uint8_t* ptr, bool mn_major, int64_t mn, int64_t K, int64_t ld,
                             int box_rows, bool bf16 = false) {
  auto enc = get_encode();
  if (!enc) return false;
  const int es = bf16 ? 2 : 1;
  const cuuint32_t inner = 128 / es;
  cuuint64_t dims[2] = {(cuuint64_t)(mn_major ? mn : K), (cuuint64_t)(mn_major ? K : mn)};
  cuuint64_t strides[1] = {(cuuint64_t)ld * es};
  cuuint32_t box[2] = {inner, (cuuint32_t)(mn_major ? BK : box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 2,
                   const_cast<uint8_t*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static int num_sms() { return device_sm_count(); }

// CTA-pair mode for the plain FP8 kinds; knob gemm_cta_group = 1 forces single-CTA tiles
// (used by the tests to cover both code paths).
static int cta_group_for() { return knob(KNOB_GEMM_CTA_GROUP) == 1 ? 1 : 2; }

// E8M0 blocked scale buffer of an MX operand with `rows` rows viewed as a 2-D u32 tensor
// [rows/128 * K/128 tiles][128 words]; a box of KS consecutive tiles = KS K atoms.
static bool make_sf_map(CUtensorMap* m, const void* ptr, int64_t rows, int64_t K, int ks) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {128, (cuuint64_t)((rows / 128) * (K / 128))};
  cuuint64_t strides[1] = {512};
  cuuint32_t box[2] = {128, (cuuint32_t)ks};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool MX, int CG, int ST, int KS, bool BF, bool GRP, bool E8, int BNT>
static bool setup_prob(const GemmProblem& p, Prob& P, CUtensorMap maps[5]) {
  // grouped 1: B holds G experts (K-major: G*N rows; MN-major: G*K contraction rows)
  const int64_t bN = p.grouped == 1 && !p.b_mn ? p.G * p.N : p.N;
  const int64_t bK = p.grouped == 1 && p.b_mn ? p.G * p.K : p.K;
  if (!make_operand_map(&maps[0], p.A, p.a_mn, p.M, p.K, p.lda, BM, BF) ||
      !make_operand_map(&maps[1], p.B, p.b_mn, bN, bK, p.ldb, BNT / CG, BF))
    return false;
  if (MX) {
    if (!make_sf_map(&maps[2], p.sa, p.M, p.K, KS) || !make_sf_map(&maps[3], p.sb, p.N, p.K, KS)) return false;
  } else {
    maps[2] = maps[0];   // unused by the plain FP8 kinds
    maps[3] = maps[1];
  }
  maps[4] = maps[0];
  const bool d_tma = (BNT == 512 || knob(KNOB_GEMM_EPI_TMA) == 1) && !p.out_f32 && !p.rs_bufs && !p.grouped &&
                     p.ldd % 8 == 0 && (reinterpret_cast<uintptr_t>(p.D) & 15) == 0;
  if (d_tma) {   // D bf16 [M, N] (row stride ldd), boxes of 32 rows x 32 columns, SWIZZLE_64B
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)p.N, (cuuint64_t)p.M};
    cuuint64_t strides[1] = {(cuuint64_t)p.ldd * 2};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t estr[2] = {1, 1};
    if (enc(&maps[4], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p.D, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  P = Prob{};
  P.M = (int)p.M; P.N = (int)p.N; P.K = (int)p.K;
  P.tiles_m = (int)((p.M + BM * CG - 1) / (BM * CG));
  P.tiles_n = (int)((p.N + BNT - 1) / BNT);
  const int k_per_stage = BF ? KS * 64 : KS * BK;   // elements
  P.num_kb = (int)((p.K + k_per_stage - 1) / k_per_stage);
  P.idesc = MX   ? make_idesc_mxf8f6f4(p.fmt_a, p.fmt_b, BM * CG, BNT, p.a_mn ? 1u : 0u, p.b_mn ? 1u : 0u)
            : BF ? make_idesc_bf16(BM * CG, BN, p.a_mn ? 1u : 0u, p.b_mn ? 1u : 0u)
                 : make_idesc_f8f6f4(p.fmt_a, p.fmt_b, BM * CG, BN, p.a_mn ? 1u : 0u, p.b_mn ? 1u : 0u);
  P.a_mn = p.a_mn;
  P.b_mn = p.b_mn;
  if (MX) {
    P.sf_tiles_k = (int)(p.K / 128);
  } else {
    P.sa = static_cast<const float*>(p.sa);
    P.sb = static_cast<const float*>(p.sb);
    P.row_scales = p.scale_mode == 1;
  }
  P.D = p.D; P.ldd = p.ldd; P.out_f32 = p.out_f32;
  P.d_tma = d_tma ? 1 : 0;
  P.out_amax = p.out_amax;
  P.grouped = p.grouped;
  P.G = p.G;
  P.offs = p.offs;
  P.chunk_done = p.chunk_done;
  P.chunk_rows = p.chunk_rows;
  P.mrot = p.mrot;
  P.chunk_epoch = p.chunk_epoch;
  P.rs_bufs = p.rs_bufs;
  P.rs_sigs = p.rs_sigs;
  P.rs_cnt = p.rs_cnt;
  P.rs_rank = p.rs_rank;
  P.rs_chunk_rows = p.rs_chunk_rows;
  // every epilogue warp of both CTAs of a pair arrives once per tile of the chunk
  P.rs_expect = p.rs_bufs ? (p.rs_chunk_rows / (BM * CG)) * P.tiles_n * Layout<MX, CG, ST, KS, BF, GRP, E8, BNT>::EPI_WARPS * CG : 0;
  P.rs_epoch = p.rs_epoch;
  return true;
}

// Tile raster of one problem: groups of GROUP_M M tiles sweep the N tiles, so the ~74 concurrent tiles
// of a wave cover 16 M x ~4.6 N tiles and share their K slices of A and B while they are read (the L2
// de-duplicates concurrent reads; the operand traffic per flop is what bounds the GEMM at full clock,
// DESIGN.md §5).  Measured (bench, 1.97 GHz): c2 step GEMMs 1.963 ms row-major -> 1.925 ms (16); 8: 1.939,
// 32: 2.02, 64: 2.16; c4 8.42-8.47 ms (8, 16) vs 9.09 (32), 9.78 (64); c3 layer step -1 to -3 %.
// (Round r01c chose row-major when all of B fit ~80 MB of L2; with the dynamic scheduler the grouped
// raster is as good or better for every shape measured.)  knob gemm_raster overrides (0 = row-major).
// Round r02 (K-serpentine on, tools/prof_raster.sh): long-K problems (K >= 16384: the c4 backward's dX and
// dW, the c2 / c5 dW) keep fewer M tiles per group -- a wave then touches ~8 A panels and ~9 B panels
// instead of 16 + 4.6, whose K slices the next wave re-reads from L2: c4 backward DRAM reads 8.35 -> 7.41 GB
// per launch and the c4 step 9.27 -> 9.07 ms; the c4 forward (K = 8192) keeps 16 (its DRAM reads 1.30 GB
// with 16 vs 2.14 GB with 8).
static int choose_raster(const GemmProblem& p, bool) { return p.K >= 16384 ? 8 : GROUP_M; }

// This launch's slot of g_sched on the current device: eager launches round-robin over
// [0, SCHED_SLOTS); a launch under stream capture takes the next unused slot of the graph region,
// which is never recycled -- once it is used up (SCHED_SLOTS captured GEMMs on this device),
// *exhausted is set and the caller falls back to the static round-robin schedule, so two graph
// nodes never share a counter.  One captured node keeps its slot for every replay: replays of the
// same graph (or of two execs instantiated from it) must not run concurrently (fp8train.h).
static unsigned* sched_slot(cudaStream_t st, bool* exhausted) {
  static std::atomic<unsigned*> base[MAX_DEVICES];
  static std::atomic<unsigned> next_slot[MAX_DEVICES], next_graph_slot[MAX_DEVICES];
  *exhausted = false;
  int dev = 0;
  if (current_device(&dev) != cudaSuccess || dev >= MAX_DEVICES) return nullptr;
  unsigned* b = base[dev].load();
  if (!b) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_sched) != cudaSuccess) return nullptr;
    b = static_cast<unsigned*>(p);
    base[dev].store(b);
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) return nullptr;
  if (cs == cudaStreamCaptureStatusActive) {
    const unsigned g = next_graph_slot[dev].fetch_add(1);
    if (g >= (unsigned)SCHED_SLOTS) {
      *exhausted = true;
      return nullptr;
    }
    return b + 2 * (SCHED_SLOTS + g);
  }
  return b + 2 * (next_slot[dev].fetch_add(1) % SCHED_SLOTS);
}

template <bool MX, int CG, int ST, int KS, bool BF = false, bool GRP = false, bool E8 = false, int BNT = 256>
static cudaError_t launch_t(const GemmProblem* ps, int n, cudaStream_t st) {
  using L = Layout<MX, CG, ST, KS, BF, GRP, E8, BNT>;
  const cudaError_t attr_err = ensure_smem<fp8_gemm_kernel<MX, CG, ST, KS, BF, GRP, E8, BNT>>(L::bytes);
  if (attr_err != cudaSuccess) return attr_err;
  if (n < 1 || n > MAXP || (GRP && n > 2)) return cudaErrorInvalidValue;
  static_assert(sizeof(GemmMaps) + sizeof(GemmArgs) <= 32000, "kernel parameter space");
  GemmMaps maps;
  GemmArgs a{};
  // longer-K problems first (stable): the dynamic scheduler then hands out the long tiles before the short ones
  GemmProblem q[MAXP];
  for (int i = 0; i < n; ++i) q[i] = ps[i];
  if (!GRP)
    std::stable_sort(q, q + n, [](const GemmProblem& x, const GemmProblem& y) { return x.K > y.K; });
  ps = q;
  a.np = n;
  a.tstart[0] = 0;
  for (int i = 0; i < n; ++i) {
    if (!setup_prob<MX, CG, ST, KS, BF, GRP, E8, BNT>(ps[i], a.p[i], maps.m[i])) return cudaErrorInvalidValue;
    a.tstart[i + 1] = a.tstart[i] + a.p[i].tiles_m * a.p[i].tiles_n;
  }
  for (int i = n; i <= MAXP; ++i) a.tstart[i] = a.tstart[n];
  a.num_tiles = a.tstart[n];
  {
    a.debug = knob(KNOB_GEMM_DEBUG);
    // knob gemm_sched = 0: round-robin tiles (A/B); default: dynamic scheduler.  A launch under
    // stream capture whose graph slot region is exhausted also takes the static schedule (no slot
    // is ever shared by two graph nodes).
    if (knob(KNOB_GEMM_SCHED) == 1) {
      bool exhausted = false;
      a.sched = sched_slot(st, &exhausted);
      if (!a.sched && !exhausted) return cudaErrorInvalidValue;
    }
    a.sf_split = knob(KNOB_MX_SF_SPLIT);
    a.kserp = knob(KNOB_GEMM_KSERP);
    a.l2pf = knob(KNOB_GEMM_L2PF);
    a.st_ef = knob(KNOB_GEMM_ST_EF);
    a.wsleep = knob(KNOB_WAIT_SLEEP);
    a.l2hint = knob(KNOB_GEMM_L2HINT);
    a.afill = knob(KNOB_GEMM_AFILL);
    bool need_fault = GRP;
    for (int i = 0; i < n; ++i) need_fault = need_fault || ps[i].chunk_done != nullptr;
    if (need_fault) {
      a.fault = fault_word(st);
      a.watchdog_ns = watchdog_ns();
    }
    // raster per problem (choose_raster); knob gemm_raster >= 0 overrides for every problem
    const int r = knob(KNOB_GEMM_RASTER);
    for (int i = 0; i < n; ++i) a.p[i].raster = r >= 0 ? r : choose_raster(ps[i], BF);
  }
  const int slots = num_sms() / CG;
  // grouped: the tile count depends on the device-side offsets -> a full persistent grid
  const int grid = GRP ? CG * slots : CG * (a.num_tiles < slots ? a.num_tiles : slots);
  LaunchScope ls(MX ? K_GEMM_MX : (BF ? K_GEMM_BF16 : K_GEMM), st);
  if (CG == 1) {
    fp8_gemm_kernel<MX, CG, ST, KS, BF, GRP, E8, BNT><<<grid, L::THREADS, L::bytes, st>>>(maps, a);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(L::THREADS);
    cfg.dynamicSmemBytes = L::bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, fp8_gemm_kernel<MX, CG, ST, KS, BF, GRP, E8, BNT>, maps, a);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

// One or two problems of the same kind (scale mode) on one persistent launch.
cudaError_t launch_gemms(const GemmProblem* ps, int n, cudaStream_t st) {
  if (n < 1 || n > MAXP) return cudaErrorInvalidValue;
  bool grp = false;
  for (int i = 0; i < n; ++i) {
    if (ps[i].grouped) {
      if (ps[i].scale_mode == 2 || ps[i].bf16_in || !ps[i].offs || ps[i].G < 1 || ps[i].G > GMAX)
        return cudaErrorInvalidValue;
      grp = true;
    }
  }
  if (grp) return launch_t<false, 2, 3, 2, false, true>(ps, n, st);
  for (int i = 1; i < n; ++i)
    if ((ps[i].scale_mode == 2) != (ps[0].scale_mode == 2)) return cudaErrorInvalidValue;
  if (ps[0].bf16_in) {
    for (int i = 1; i < n; ++i)
      if (!ps[i].bf16_in) return cudaErrorInvalidValue;
    return launch_t<false, 2, 3, 2, true>(ps, n, st);
  }
  const int cg = cta_group_for();
  if (ps[0].scale_mode == 2) {
    if (cg == 1) return launch_t<true, 1, 4, 1>(ps, n, st);
    // knob mx_n192 = 1 (K-major operands only): N = 192 tiles with double-buffered accumulators.  Measured
    // 18 % fewer flop/clk/SM than N = 256 with one accumulator (c4 shape 10.5k vs 12.8k): the extra
    // operand traffic per flop costs more than the accumulator hand-over saves.  Kept as an option.
    bool kmaj = true;
    for (int i = 0; i < n; ++i) kmaj = kmaj && !ps[i].a_mn && !ps[i].b_mn;
    if (kmaj && knob(KNOB_MX_N192) == 1) return launch_t<true, 2, 3, 2, false, false, false, 192>(ps, n, st);
    return launch_t<true, 2, 3, 2>(ps, n, st);
  }
  if (cg == 1) return launch_t<false, 1, 4, 1>(ps, n, st);
  // 256 x 512 tiles (knob gemm_n512) when every problem's N is a multiple of 512: 4 stages x 1 atom
  // (48 KB per CTA per stage: A 16 KB + B 32 KB) + 4 KB of TMA-store output chunks per epilogue warp
  // knob 1: whenever the shapes allow; 2 (auto): only when every problem also has K >= 8192 -- the single
  // accumulator's per-tile hand-over costs more than the operand savings on short-K tiles (c3's wq/wk/wv/wo
  // backward: -5 %), long-K launches gain 1-3 % (round-2 A/B)
  const int n512 = knob(KNOB_GEMM_N512);
  if (n512 && knob(KNOB_GEMM_STAGES) == 3) {
    bool ok = true;
    for (int i = 0; i < n; ++i) ok = ok && ps[i].N % 512 == 0 && !ps[i].grouped && (n512 == 1 || ps[i].K >= 8192);
    if (ok) return launch_t<false, 2, 4, 1, false, false, false, 512>(ps, n, st);
  }
  // default: 3 stages x 2 K atoms (64 KB per CTA per stage, 8 MMAs per barrier round trip);
  // knob gemm_stages = 6 selects 6 x 1 atom (4 MMAs per round trip) for comparison
  const int stages = knob(KNOB_GEMM_STAGES);
  if (stages == 6) return launch_t<false, 2, 6, 1>(ps, n, st);
  if (stages == 4) return launch_t<false, 2, 4, 1>(ps, n, st);
  // short-K launches (tiles of <= 1024-deep K) are epilogue-bound: 8 epilogue warps (measured: K = 1024
  // 7.5k -> 8.6k flop/clk/SM; K = 2048 10.6k with 4 warps vs 9.9k with 8)
  bool short_k = false;
  for (int i = 0; i < n; ++i) short_k = short_k || ps[i].K <= 1024;
  const int epi = knob(KNOB_GEMM_EPI);
  if (epi) short_k = epi == 8;
  return short_k ? launch_t<false, 2, 3, 2, false, false, true>(ps, n, st) : launch_t<false, 2, 3, 2>(ps, n, st);
}

cudaError_t launch_gemm(const GemmProblem& p, cudaStream_t st) { return launch_gemms(&p, 1, st); }

}  // namespace fp8t
