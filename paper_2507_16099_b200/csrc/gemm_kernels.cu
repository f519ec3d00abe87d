// Scaled FP8 GEMM on 5th-generation tensor cores (tcgen05), sm_100a.
//
//   D[m,n] = sum_k dec(A[m,k]) dec(B[n,k]) * epilogue scales
//
// Persistent, warp-specialised, one CTA per SM:
//   warp 0      TMA producer: A/B tiles (SWIZZLE_128B) into a 4-stage smem ring; MX: E8M0
//               scale-factor tiles by 1-D bulk copy
//   warp 1      MMA issuer: one thread issues tcgen05.mma.kind::f8f6f4 (or
//               kind::mxf8f6f4.block_scale) 128x256x32 per instruction into a TMEM
//               accumulator; tcgen05.commit frees smem stages / publishes accumulators
//   warp 2      TMEM allocator
//   warps 4..7  epilogue: tcgen05.ld 32 lanes x 32 columns -> fp32 -> * (1/sa)(1/sb) ->
//               bf16/fp32 -> global
// Accumulators are double-buffered in TMEM (2 x 256 columns) for the plain FP8 kinds so
// the epilogue of tile i overlaps the mainloop of tile i+1; the MX kind keeps one
// accumulator (256 columns) plus the scale-factor columns.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <mutex>

#include "kernels.h"
#include "ptx.cuh"

namespace fp8t {

constexpr int BM = 128, BN = 256, BK = 128, STAGES = 4;
constexpr int A_STAGE = BM * BK;        // 16 KB
constexpr int B_STAGE = BN * BK;        // 32 KB
constexpr int SFA_STAGE = 512;          // 128 rows x 4 K-blocks of E8M0
constexpr int SFB_STAGE = 1024;         // 256 rows x 4
constexpr int GROUP_M = 16;             // tile raster: 16 M-tiles share the N sweep (L2 reuse)

struct GemmArgs {
  int M, N, K;
  int tiles_m, tiles_n, num_tiles, num_kb;
  uint32_t idesc;
  const float* sa; const float* sb;
  const uint8_t* sfa; const uint8_t* sfb;
  int sf_tiles_k;     // K / 128: 512-byte scale tiles per 128-row block
  void* D; int64_t ldd; int out_f32; int row_scales;
};

template <bool MX> struct Layout {
  static constexpr int ACC = MX ? 1 : 2;
  static constexpr uint32_t off_a = 0;
  static constexpr uint32_t off_b = off_a + STAGES * A_STAGE;
  static constexpr uint32_t off_sfa = off_b + STAGES * B_STAGE;
  static constexpr uint32_t off_sfb = off_sfa + (MX ? STAGES * SFA_STAGE : 0);
  static constexpr uint32_t off_bar = off_sfb + (MX ? STAGES * SFB_STAGE : 0);
  static constexpr uint32_t n_bar = 2 * STAGES + 2 * ACC;
  static constexpr uint32_t off_tmem = off_bar + 8 * n_bar;
  static constexpr uint32_t bytes = off_tmem + 16 + 1024;  // + alignment slack
  static constexpr uint32_t tmem_cols = 512;
  static constexpr uint32_t sfa_col = 256, sfb_col = 260;  // MX only (after one accumulator)
};

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int& mb, int& nb) {
  const int group = t / (GROUP_M * tiles_n);
  const int first_m = group * GROUP_M;
  const int gsz = min(GROUP_M, tiles_m - first_m);
  const int local = t - group * GROUP_M * tiles_n;
  mb = first_m + local % gsz;
  nb = local / gsz;
}

template <bool MX>
__global__ void __launch_bounds__(256, 1)
    fp8_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const GemmArgs args) {
  using L = Layout<MX>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t full_bar = base + L::off_bar;                 // [STAGES]
  const uint32_t empty_bar = full_bar + 8 * STAGES;            // [STAGES]
  const uint32_t tfull_bar = empty_bar + 8 * STAGES;           // [ACC]
  const uint32_t tempty_bar = tfull_bar + 8 * L::ACC;          // [ACC]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + L::off_tmem);

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar + 8 * s, 1);
      mbar_init(empty_bar + 8 * s, 1);
    }
    for (int a = 0; a < L::ACC; ++a) {
      mbar_init(tfull_bar + 8 * a, 1);
      mbar_init(tempty_bar + 8 * a, 128);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc(smem_u32(tmem_slot), L::tmem_cols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < args.num_tiles; tile += gridDim.x) {
      int mb, nb;
      tile_coords(tile, args.tiles_m, args.tiles_n, mb, nb);
      const bool sfb_hi = MX && (2 * nb + 1) * 128 < args.N;
      const uint32_t tx = A_STAGE + B_STAGE + (MX ? SFA_STAGE + (sfb_hi ? SFB_STAGE : SFB_STAGE / 2) : 0);
      for (int kb = 0; kb < args.num_kb; ++kb) {
        mbar_wait(empty_bar + 8 * stage, phase ^ 1);
        if (lane == 0) {
          const uint32_t fb = full_bar + 8 * stage;
          mbar_arrive_expect_tx(fb, tx);
          tma_load_2d(base + L::off_a + stage * A_STAGE, &tmA, kb * BK, mb * BM, fb, 0);
          tma_load_2d(base + L::off_b + stage * B_STAGE, &tmB, kb * BK, nb * BN, fb, 0);
          if (MX) {
            const uint8_t* sa = args.sfa + ((int64_t)mb * args.sf_tiles_k + kb) * 512;
            const uint8_t* sb = args.sfb + ((int64_t)(2 * nb) * args.sf_tiles_k + kb) * 512;
            bulk_load(base + L::off_sfa + stage * SFA_STAGE, sa, 512, fb);
            bulk_load(base + L::off_sfb + stage * SFB_STAGE, sb, 512, fb);
            if (sfb_hi) bulk_load(base + L::off_sfb + stage * SFB_STAGE + 512, sb + (int64_t)args.sf_tiles_k * 512, 512, fb);
          }
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < args.num_tiles; tile += gridDim.x) {
      mbar_wait(tempty_bar + 8 * acc, acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < args.num_kb; ++kb) {
        mbar_wait(full_bar + 8 * stage, phase);
        tc_fence_after();
        if (lane == 0) {
          if (MX) {
            tmem_cp_32x128b_warpx4(tmem_base + L::sfa_col, make_sf_desc(base + L::off_sfa + stage * SFA_STAGE));
            tmem_cp_32x128b_warpx4(tmem_base + L::sfb_col, make_sf_desc(base + L::off_sfb + stage * SFB_STAGE));
            tmem_cp_32x128b_warpx4(tmem_base + L::sfb_col + 4,
                                   make_sf_desc(base + L::off_sfb + stage * SFB_STAGE + 512));
          }
          const uint64_t adesc = make_sw128_kmajor_desc(base + L::off_a + stage * A_STAGE);
          const uint64_t bdesc = make_sw128_kmajor_desc(base + L::off_b + stage * B_STAGE);
#pragma unroll
          for (int k = 0; k < BK / 32; ++k) {
            // advance 32 bytes along K inside the 128-byte swizzle atom (start address >> 4)
            const uint64_t koff = (uint64_t)(k * 32 >> 4);
            if (MX)
              mma_mxf8f6f4(d_tmem, adesc + koff, bdesc + koff, idesc_with_sf_id(args.idesc, k, k),
                           (kb | k) != 0, tmem_base + L::sfa_col, tmem_base + L::sfb_col);
            else
              mma_f8f6f4(d_tmem, adesc + koff, bdesc + koff, args.idesc, (kb | k) != 0);
          }
          mma_commit(empty_bar + 8 * stage);
          if (kb == args.num_kb - 1) mma_commit(tfull_bar + 8 * acc);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (++acc == L::ACC) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    float ts = 1.f;
    if (!args.row_scales && args.sa) ts = __frcp_rn(args.sa[0]) * __frcp_rn(args.sb[0]);
    for (int tile = blockIdx.x; tile < args.num_tiles; tile += gridDim.x) {
      int mb, nb;
      tile_coords(tile, args.tiles_m, args.tiles_n, mb, nb);
      const int row = mb * BM + q * 32 + (int)lane;
      const bool rvalid = row < args.M;
      float rs = ts;
      if (args.row_scales && rvalid) rs = __frcp_rn(args.sa[row]);
      mbar_wait(tfull_bar + 8 * acc, acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, r);
        tmem_wait_ld();
        const int col0 = nb * BN + c * 32;
        if (!rvalid || col0 >= args.N) continue;
        float v[32];
        if (args.row_scales) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int col = min(col0 + j, args.N - 1);
            v[j] = __fmul_rn(__fmul_rn(__uint_as_float(r[j]), rs), __frcp_rn(args.sb[col]));
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __fmul_rn(__uint_as_float(r[j]), rs);
        }
        const int nvalid = min(32, args.N - col0);  // 16 or 32 (N % 16 == 0)
        if (args.out_f32) {
          float* dst = reinterpret_cast<float*>(args.D) + (int64_t)row * args.ldd + col0;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (4 * j < nvalid) reinterpret_cast<float4*>(dst)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        } else {
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
            pk[j] = *reinterpret_cast<uint32_t*>(&h);
          }
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(args.D) + (int64_t)row * args.ldd + col0;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (8 * j < nvalid) reinterpret_cast<uint4*>(dst)[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(tempty_bar + 8 * acc);
      if (++acc == L::ACC) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, L::tmem_cols);
  }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
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

static bool make_kmajor_map(CUtensorMap* m, const uint8_t* ptr, int64_t rows, int64_t K, int64_t ld, int box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <bool MX>
static cudaError_t launch_t(const GemmProblem& p, cudaStream_t st) {
  using L = Layout<MX>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(fp8_gemm_kernel<MX>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::bytes);
  });
  if (attr_err != cudaSuccess) return attr_err;
  CUtensorMap ta, tb;
  if (!make_kmajor_map(&ta, p.A, p.M, p.K, p.lda, BM) || !make_kmajor_map(&tb, p.B, p.N, p.K, p.ldb, BN))
    return cudaErrorInvalidValue;
  GemmArgs a{};
  a.M = (int)p.M; a.N = (int)p.N; a.K = (int)p.K;
  a.tiles_m = (int)((p.M + BM - 1) / BM);
  a.tiles_n = (int)((p.N + BN - 1) / BN);
  a.num_tiles = a.tiles_m * a.tiles_n;
  a.num_kb = (int)((p.K + BK - 1) / BK);
  a.idesc = MX ? make_idesc_mxf8f6f4(p.fmt_a, p.fmt_b, BM, BN) : make_idesc_f8f6f4(p.fmt_a, p.fmt_b, BM, BN);
  if (MX) {
    a.sfa = static_cast<const uint8_t*>(p.sa);
    a.sfb = static_cast<const uint8_t*>(p.sb);
    a.sf_tiles_k = (int)(p.K / 128);
  } else {
    a.sa = static_cast<const float*>(p.sa);
    a.sb = static_cast<const float*>(p.sb);
    a.row_scales = p.scale_mode == 1;
  }
  a.D = p.D; a.ldd = p.ldd; a.out_f32 = p.out_f32;
  const int grid = a.num_tiles < num_sms() ? a.num_tiles : num_sms();
  LaunchScope ls(MX ? K_GEMM_MX : K_GEMM, st);
  fp8_gemm_kernel<MX><<<grid, 256, L::bytes, st>>>(ta, tb, a);
  return cudaGetLastError();
}

cudaError_t launch_gemm(const GemmProblem& p, cudaStream_t st) {
  return p.scale_mode == 2 ? launch_t<true>(p, st) : launch_t<false>(p, st);
}

}  // namespace fp8t
