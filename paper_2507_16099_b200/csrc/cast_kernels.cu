// Memory-bound kernels of the Float8Linear step (HBM roofline):
//   amax_tile   : max|x| per tensor / row / column  (Appendix A)
//   cast_tile   : s = RN32(fmax/max(amax,eps)); q = satRNE(RN32(x*s)); row-major and/or
//                 transposed FP8 output from one read (tensorwise / rowwise casts)
//   mx_cast     : MXFP8 dim0 + dim1 casts with E8M0 block-32 scales from one read
//   transpose_u8: FP8 byte transpose (pre-gathered FSDP weight -> the dX operand)
// All kernels read 128 x 128 tiles with 16-byte vector loads; transposed outputs go
// through a 16 KB XOR-swizzled shared-memory tile and leave as 16-byte stores.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>

#include "kernels.h"
#include "ptx.cuh"
#include "scale.cuh"

namespace fp8t {


// ---------------------------------------------------------------------------
// 8-element loads as fp32 (exact widening) and |x| bit patterns
// ---------------------------------------------------------------------------
template <typename T> struct Ld8;
template <> struct Ld8<float> {
  static __device__ __forceinline__ void load(const float* p, float (&v)[8]) {
    float4 a = __ldg(reinterpret_cast<const float4*>(p));
    float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
};
template <> struct Ld8<__nv_bfloat16> {
  static __device__ __forceinline__ void load(const __nv_bfloat16* p, float (&v)[8]) {
    uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
};
// Raw (undecoded) 8-element loads: issue all of a tile's loads before decoding so each
// thread keeps 8 independent 16-32 B requests in flight with few registers.
template <typename T> struct Raw8;
template <> struct Raw8<float> {
  float4 a, b;
  __device__ __forceinline__ void load(const float* p) {
    a = __ldg(reinterpret_cast<const float4*>(p));
    b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  }
  __device__ __forceinline__ void zero() { a = b = make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ __forceinline__ void get(float (&v)[8]) const {
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
};
template <> struct Raw8<__nv_bfloat16> {
  uint4 u;
  __device__ __forceinline__ void load(const __nv_bfloat16* p) { u = __ldg(reinterpret_cast<const uint4*>(p)); }
  __device__ __forceinline__ void zero() { u = make_uint4(0, 0, 0, 0); }
  __device__ __forceinline__ void get(float (&v)[8]) const {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
};

__device__ __forceinline__ int imin128(int64_t v) { return v < 128 ? (int)v : 128; }

// Segment of row r0 (grouped recipe): returns its index and first row.  offs: the g with
// offs[g] <= r0 < offs[g+1] (empty groups skipped); seg_rows: fixed-size segments.
__device__ __forceinline__ int seg_of(const Seg& sg, int64_t r0, int64_t& start) {
  if (sg.offs) {
    int lo = 0, hi = sg.G;   // invariant: offs[lo] <= r0 < offs[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(sg.offs + mid) <= r0) lo = mid; else hi = mid;
    }
    start = __ldg(sg.offs + lo);
    return lo;
  }
  if (sg.seg_rows > 0) {
    const int g = (int)(r0 / sg.seg_rows);
    start = (int64_t)g * sg.seg_rows;
    return g;
  }
  start = 0;
  return 0;
}
__device__ __forceinline__ uint32_t abs_bits(float v) { return __float_as_uint(v) & 0x7FFFFFFFu; }

// x * s rounded to fp32 (IEEE RN, R-c4) two lanes per instruction (__fmul2_rn), then satRNE to FP8.
template <int FMT>
__device__ __forceinline__ uint2 cast8(const float (&v)[8], float s) {
  float p[8];
#pragma unroll
  for (int i = 0; i < 8; i += 2) {
    const float2 q = __fmul2_rn(make_float2(v[i], v[i + 1]), make_float2(s, s));
    p[i] = q.x;
    p[i + 1] = q.y;
  }
  return make_uint2(cvt_x4<FMT>(p[0], p[1], p[2], p[3]), cvt_x4<FMT>(p[4], p[5], p[6], p[7]));
}
template <int FMT>
__device__ __forceinline__ uint2 cast8v(const float (&v)[8], const float* s) {
  float p[8];
#pragma unroll
  for (int i = 0; i < 8; i += 2) {
    const float2 q = __fmul2_rn(make_float2(v[i], v[i + 1]), make_float2(s[i], s[i + 1]));
    p[i] = q.x;
    p[i + 1] = q.y;
  }
  return make_uint2(cvt_x4<FMT>(p[0], p[1], p[2], p[3]), cvt_x4<FMT>(p[4], p[5], p[6], p[7]));
}

// ---------------------------------------------------------------------------
// Transposed-tile staging.  Tile = 128 rows x 128 bytes; word w of row r lives at
// word position w ^ (((r >> 4) & 7) << 2), which makes both the row-wise writes
// and the 16-row column reads below bank-conflict free.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int swz(int r, int w) { return r * 32 + (w ^ (((r >> 4) & 7) << 2)); }

// 4x4 byte transpose: in a,b,c,d = rows (4 column bytes each) -> out[j] = column j (4 row bytes).
__device__ __forceinline__ void transpose4x4(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t (&o)[4]) {
  uint32_t t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(a, b, 0x7362);
  uint32_t t2 = __byte_perm(c, d, 0x5140), t3 = __byte_perm(c, d, 0x7362);
  o[0] = __byte_perm(t0, t2, 0x5410);
  o[1] = __byte_perm(t0, t2, 0x7632);
  o[2] = __byte_perm(t1, t3, 0x5410);
  o[3] = __byte_perm(t1, t3, 0x7632);
}

// Phase 2: each thread reads a 16-row x 4-column block of the staged tile and writes
// the 4 transposed rows (16 bytes each).  Threads t..t+7 cover 128 contiguous bytes.
__device__ __forceinline__ void store_transposed(const uint32_t* tile, uint8_t* qt, int64_t ldt, int64_t r0,
                                                 int64_t c0, int vrows, int vcols) {
  const int t = threadIdx.x;
  const int rg = t & 7, w = t >> 3;
  if (16 * rg >= vrows || 4 * w >= vcols) return;
  uint32_t W[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) W[i] = tile[swz(16 * rg + i, w)];
  uint32_t o[4][4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    uint32_t col[4];
    transpose4x4(W[4 * g], W[4 * g + 1], W[4 * g + 2], W[4 * g + 3], col);
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j][g] = col[j];
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint8_t* dst = qt + (c0 + 4 * w + j) * ldt + r0 + 16 * rg;
    *reinterpret_cast<uint4*>(dst) = make_uint4(o[j][0], o[j][1], o[j][2], o[j][3]);
  }
}

// ---------------------------------------------------------------------------
// amax over a 128 x 128 tile: tensor / per-row / per-column maxima, merged with
// u32 atomicMax on |x| bit patterns (exact, order independent).  Output buffers
// must be zeroed beforehand.
// ---------------------------------------------------------------------------
template <typename T, int MODE>  // MODE bit0: tensor, bit1: row, bit2: col
__global__ void __launch_bounds__(256) amax_tile_kernel(const T* __restrict__ x, int64_t R, int64_t C, int64_t ld,
                                                        uint32_t* amax_tensor, uint32_t* amax_row,
                                                        uint32_t* amax_col, const Seg seg) {
  // Persistent over 128 x 128 tiles in increasing linear order (the cast kernel walks them in
  // decreasing order, so its first reads hit the tiles this kernel touched last, still in L2).
  __shared__ uint32_t colred[8][128];
  __shared__ uint32_t wred[8];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int tiles_x = (int)((C + 127) >> 7);
  const int num_tiles = tiles_x * (int)((R + 127) >> 7);
  const int cc = (t & 15) * 8;
  uint32_t tmax = 0;
  for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
    const int64_t r0 = (int64_t)(tile / tiles_x) * 128, c0 = (int64_t)(tile % tiles_x) * 128;
    const bool cvalid = c0 + cc < C;
    uint32_t cmax[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    Raw8<T> raw[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t r = r0 + (t >> 4) + 16 * i;
      if (cvalid && r < R) raw[i].load(x + r * ld + c0 + cc);
      else raw[i].zero();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t rmax = 0;
      float vi[8];
      raw[i].get(vi);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t a = abs_bits(vi[e]);
        rmax = max(rmax, a);
        cmax[e] = max(cmax[e], a);
      }
      tmax = max(tmax, rmax);
      if (MODE & 2) {
        rmax = max(rmax, __shfl_xor_sync(0xffffffffu, rmax, 1));
        rmax = max(rmax, __shfl_xor_sync(0xffffffffu, rmax, 2));
        rmax = max(rmax, __shfl_xor_sync(0xffffffffu, rmax, 4));
        rmax = max(rmax, __shfl_xor_sync(0xffffffffu, rmax, 8));
        const int64_t r = r0 + (t >> 4) + 16 * i;
        if ((t & 15) == 0 && r < R) atomicMax(amax_row + r, rmax);
      }
    }
    if (MODE & 4) {
#pragma unroll
      for (int e = 0; e < 8; ++e) cmax[e] = max(cmax[e], __shfl_xor_sync(0xffffffffu, cmax[e], 16));
      if (lane < 16) {
#pragma unroll
        for (int e = 0; e < 8; ++e) colred[warp][cc + e] = cmax[e];
      }
      __syncthreads();
      if (t < 128 && c0 + t < C) {
        uint32_t m = colred[0][t];
#pragma unroll
        for (int w = 1; w < 8; ++w) m = max(m, colred[w][t]);
        int64_t sstart;
        const int g = seg_of(seg, r0, sstart);
        atomicMax(amax_col + (int64_t)g * C + c0 + t, m);
      }
      __syncthreads();
    }
  }
  if (MODE & 1) {  // one atomic per CTA for the tensor amax
    tmax = __reduce_max_sync(0xffffffffu, tmax);
    if (lane == 0) wred[warp] = tmax;
    __syncthreads();
    if (t == 0) {
      uint32_t m = wred[0];
#pragma unroll
      for (int i = 1; i < 8; ++i) m = max(m, wred[i]);
      atomicMax(amax_tensor, m);
    }
  }
}

// ---------------------------------------------------------------------------
// amax_tile, TMA-pipelined persistent variant (bf16; rows, cols multiples of 128).  Same outputs
// as amax_tile_kernel.  CTA b owns the contiguous row-major tile range [b*per, (b+1)*per), so its
// tiles run along one or two 128-row strips: per-row maxima stay in registers across the strip
// and are flushed (half-warp reduce + one atomicMax per row) only when the strip changes, while
// thread 0 streams 32 KB tiles into an ST-deep smem ring with cp.async.bulk.tensor.
// ---------------------------------------------------------------------------
// Optional second tensor of an amax_tile_tma launch (the forward's W next to X): its tiles follow the
// first tensor's in the tile order, with their own row / column outputs (row / column modes only).
struct AmaxSecond {
  int tiles0, tiles1;  // tiles of the first / second tensor (tiles1 = 0: one tensor)
  int tiles_x1, strips0;
  uint32_t* amax_row1;
  uint32_t* amax_col1;
};

template <int MODE, int ST>
__global__ void __launch_bounds__(256) amax_tile_tma_kernel(const __grid_constant__ CUtensorMap tmap, int64_t R,
                                                            int64_t C, uint32_t* amax_tensor, uint32_t* amax_row,
                                                            uint32_t* amax_col, const Seg seg,
                                                            const __grid_constant__ CUtensorMap tmap1,
                                                            const AmaxSecond d) {
  constexpr int STAGE = 128 * 256;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint32_t(*colred)[128] = reinterpret_cast<uint32_t(*)[128]>(sm + ST * STAGE);
  uint32_t* wred = reinterpret_cast<uint32_t*>(sm + ST * STAGE + 8 * 128 * 4);
  const uint32_t bar0 = smem_u32(sm + ST * STAGE + 8 * 128 * 4 + 64), stage0 = smem_u32(sm);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int tiles_x = (int)(C >> 7);
  const int num_tiles = d.tiles0 + d.tiles1;
  const int per = (num_tiles + (int)gridDim.x - 1) / (int)gridDim.x;
  const int first = (int)blockIdx.x * per;
  const int last = min(first + per, num_tiles);
  // tile id -> (tensor k, strip key, column tile): strips of the second tensor are numbered after the first's
  auto where = [&](int id, int& k, int& rt, int& ct) {
    k = id >= d.tiles0 ? 1 : 0;
    const int local = k ? id - d.tiles0 : id;
    const int tx = k ? d.tiles_x1 : tiles_x;
    rt = local / tx;
    ct = local - rt * tx;
  };
  auto issue = [&](int k) {
    const int id = first + k;
    if (id < last) {
      int kk, rt, ct;
      where(id, kk, rt, ct);
      const uint32_t bar = bar0 + 8 * (k % ST);
      mbar_arrive_expect_tx(bar, STAGE);
      tma_load_2d(stage0 + (k % ST) * STAGE, kk ? &tmap1 : &tmap, ct * 128, rt * 128, bar, l2_policy_evict_first());
    }
  };
  if (t == 0) {
    tma_prefetch_desc(&tmap);
    if (d.tiles1) tma_prefetch_desc(&tmap1);
    for (int i = 0; i < ST; ++i) mbar_init(bar0 + 8 * i, 1);
    fence_mbar_init();
    for (int k = 0; k < ST; ++k) issue(k);
  }
  __syncthreads();
  const int cc = (t & 15) * 8;
  uint32_t tmax = 0;
  uint32_t rm[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // this thread's partial row maxima of the current strip
  // strip key: row strip of the first tensor, or strips0 + row strip of the second
  auto strip_of = [&](int id) {
    int kk, rt, ct;
    where(id, kk, rt, ct);
    return kk ? d.strips0 + rt : rt;
  };
  int strip = first < last ? strip_of(first) : -1;
  auto flush_rows = [&](int st_) {
    uint32_t* rowp = st_ >= d.strips0 ? d.amax_row1 + (int64_t)(st_ - d.strips0) * 128 : amax_row + (int64_t)st_ * 128;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t m = rm[i];
      m = max(m, __shfl_xor_sync(0xffffffffu, m, 1));
      m = max(m, __shfl_xor_sync(0xffffffffu, m, 2));
      m = max(m, __shfl_xor_sync(0xffffffffu, m, 4));
      m = max(m, __shfl_xor_sync(0xffffffffu, m, 8));
      if ((t & 15) == 0) atomicMax(rowp + (t >> 4) + 16 * i, m);
      rm[i] = 0;
    }
  };
  for (int k = 0; first + k < last; ++k) {
    const int id = first + k;
    int kk, rt, ct;
    where(id, kk, rt, ct);
    const int64_t r0 = (int64_t)rt * 128, c0 = (int64_t)ct * 128;
    const int skey = kk ? d.strips0 + rt : rt;
    if ((MODE & 2) && skey != strip) {
      flush_rows(strip);
      strip = skey;
    }
    mbar_wait(bar0 + 8 * (k % ST), (uint32_t)(k / ST) & 1u);
    uint4 raw[8];
    const uint8_t* sp = sm + (k % ST) * STAGE + (t >> 4) * 256 + cc * 2;
#pragma unroll
    for (int i = 0; i < 8; ++i) raw[i] = *reinterpret_cast<const uint4*>(sp + i * 16 * 256);
    __syncthreads();   // (1) stage consumed
    if (t == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k + ST);
    }
    uint32_t cmw[4] = {0, 0, 0, 0};   // packed column maxima (bf16 |x| bit pairs)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t a0 = raw[i].x & 0x7FFF7FFFu, a1 = raw[i].y & 0x7FFF7FFFu;
      const uint32_t a2 = raw[i].z & 0x7FFF7FFFu, a3 = raw[i].w & 0x7FFF7FFFu;
      if (MODE & 4) {
        cmw[0] = __vmaxu2(cmw[0], a0); cmw[1] = __vmaxu2(cmw[1], a1);
        cmw[2] = __vmaxu2(cmw[2], a2); cmw[3] = __vmaxu2(cmw[3], a3);
      }
      if (MODE & 3) {
        const uint32_t m2 = __vmaxu2(__vmaxu2(a0, a1), __vmaxu2(a2, a3));
        const uint32_t m = max(m2 & 0xFFFFu, m2 >> 16) << 16;
        if (MODE & 2) rm[i] = max(rm[i], m);
        else tmax = max(tmax, m);
      }
    }
    if (MODE & 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) cmw[j] = __vmaxu2(cmw[j], __shfl_xor_sync(0xffffffffu, cmw[j], 16));
      if (lane < 16) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          colred[warp][cc + 2 * j] = cmw[j] << 16;
          colred[warp][cc + 2 * j + 1] = cmw[j] & 0xFFFF0000u;
        }
      }
      __syncthreads();   // (2)
      if (t < 128) {
        uint32_t m = colred[0][t];
#pragma unroll
        for (int w = 1; w < 8; ++w) m = max(m, colred[w][t]);
        if (kk) {
          atomicMax(d.amax_col1 + c0 + t, m);
        } else {
          int64_t sstart;
          const int g = seg_of(seg, r0, sstart);
          atomicMax(amax_col + (int64_t)g * C + c0 + t, m);
        }
      }
    }
  }
  if (MODE & 2) {
    if (strip >= 0) flush_rows(strip);
    if (MODE & 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) tmax = max(tmax, rm[i]);
    }
  }
  if (MODE & 1) {
    tmax = __reduce_max_sync(0xffffffffu, tmax);
    if (lane == 0) wred[warp] = tmax;
    __syncthreads();
    if (t == 0) {
      uint32_t m = wred[0];
#pragma unroll
      for (int i = 1; i < 8; ++i) m = max(m, wred[i]);
      if (m) atomicMax(amax_tensor, m);
    }
  }
}

// ---------------------------------------------------------------------------
// amax_rc: row / column amax of up to AMAX_RC_MAX bf16 tensors in one launch (knob amax_rc; the
// product path for row / column amax).  Same outputs as amax_tile_tma_kernel, without a CTA-wide
// barrier per tile:
//   * one producer warp streams each 128 x 128 tile as two 64-column TMA boxes (SWIZZLE_128B) into an
//     ST-deep ring (full barrier: TMA bytes; empty barrier: one arrival per consumer warp);
//   * consumer warp w owns the 16 columns [16w, 16w + 16) of every tile, lane l reads 8 of them
//     (16 bytes) on rows l % 16 + 16 i -- with the 128-byte swizzle the 8 lanes of a shared-memory
//     phase hit 8 different bank groups.  A warp releases the stage right after its loads;
//   * column maxima: a 16-lane shuffle reduction per tile, then one atomicMax per column (the 8 lanes
//     of each half-warp holding the 8 columns);
//   * row maxima stay in registers while the CTA's contiguous tile range walks a 128-row strip and are
//     flushed (xor-16 shuffle + one atomicMax per row and warp) when the strip changes.
// Tensors are numbered consecutively: tiles [tstart[k], tstart[k+1]) belong to tensor k, row-major over
// its tile grid.  seg (grouped recipe) applies to tensor 0's column outputs.
// ---------------------------------------------------------------------------
template <int MODE, int ST>
__global__ void __launch_bounds__(288) amax_rc_kernel(const __grid_constant__ AmaxRCArgs a) {
  constexpr int STAGE = 128 * 256, BOX = STAGE / 2;
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  const uint32_t raw0 = smem_u32(sm_raw);
  const uint32_t base = (raw0 + 1023u) & ~1023u;   // SWIZZLE_128B boxes need 1024-byte alignment
  const uint8_t* smp = sm_raw + (base - raw0);
  const uint32_t full0 = base + ST * STAGE, empty0 = full0 + 8 * ST;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int total = a.tstart[a.n];
  const int per = (total + (int)gridDim.x - 1) / (int)gridDim.x;
  const int first = (int)blockIdx.x * per;
  const int last = min(first + per, total);
  if (t == 0) {
    for (int i = 0; i < ST; ++i) {
      mbar_init(full0 + 8 * i, 1);
      mbar_init(empty0 + 8 * i, 8);
    }
    fence_mbar_init();
  }
  __syncthreads();
  // The CTA's tiles [first, last) in row-major order over each tensor's tile grid, tensor after tensor: one
  // division to place the first tile, then a cursor (no per-tile division or search).
  struct Cursor {
    int k, rt, ct, id;
  };
  auto start = [&](int id) {
    Cursor c{0, 0, 0, id};
    while (c.k + 1 < a.n && id >= a.tstart[c.k + 1]) ++c.k;
    const int local = id - a.tstart[c.k];
    c.rt = local / a.tiles_x[c.k];
    c.ct = local - c.rt * a.tiles_x[c.k];
    return c;
  };
  auto advance = [&](Cursor& c) {
    ++c.id;
    if (++c.ct == a.tiles_x[c.k]) {
      c.ct = 0;
      ++c.rt;
    }
    if (c.k + 1 < a.n && c.id == a.tstart[c.k + 1]) {
      ++c.k;
      c.rt = 0;
      c.ct = 0;
    }
  };
  if (warp == 8) {   // producer
    if (lane == 0) {
      for (int i = 0; i < a.n; ++i) tma_prefetch_desc(&a.map[i]);
      const uint64_t pol = l2_policy_evict_first();
      Cursor cur = start(first);
      for (int k = 0; first + k < last; ++k, advance(cur)) {
        const int s = k % ST;
        if (k >= ST) {
          mbar_wait_opt(empty0 + 8 * s, (uint32_t)(k / ST - 1) & 1u, a.sleep);
          fence_proxy_async_smem();
        }
        const int kk = cur.k, rt = cur.rt, ct = cur.ct;
        mbar_arrive_expect_tx(full0 + 8 * s, STAGE);
        tma_load_2d(base + s * STAGE, &a.map[kk], ct * 128, rt * 128, full0 + 8 * s, pol);
        tma_load_2d(base + s * STAGE + BOX, &a.map[kk], ct * 128 + 64, rt * 128, full0 + 8 * s, pol);
      }
    }
    return;
  }
  const int r16 = lane & 15;
  const int ch = (warp & 3) * 2 + (lane >> 4);   // 16-byte chunk of the 128-byte box row
  const uint32_t off = (uint32_t)(warp >> 2) * BOX + r16 * 128 + ((ch ^ (r16 & 7)) << 4);
  const int colw = (warp >> 2) * 64 + (warp & 3) * 16 + (lane >> 4) * 8;   // first column of the thread's 8
  uint32_t rm[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int strip = -1, fk = 0, frt = 0;
  auto flush_rows = [&]() {
    uint32_t* rowp = a.row[fk] + (int64_t)frt * 128;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t m = max(rm[i], __shfl_xor_sync(0xffffffffu, rm[i], 16));
      if (lane < 16 && m) atomicMax(rowp + lane + 16 * i, m);
      rm[i] = 0;
    }
  };
  if (a.dbg & 1) {   // A/B only: consume nothing (the TMA stream alone), results invalid
    for (int k = 0; first + k < last; ++k) {
      const int s = k % ST;
      mbar_wait_opt(full0 + 8 * s, (uint32_t)(k / ST) & 1u, a.sleep);
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8 * s);
    }
    return;
  }
  Cursor cur = start(first);
  for (int k = 0; first + k < last; ++k, advance(cur)) {
    const int kk = cur.k, rt = cur.rt, ct = cur.ct;
    if (MODE & 2) {
      const int skey = a.strip0[kk] + rt;
      if (skey != strip) {
        if (strip >= 0) flush_rows();
        strip = skey;
        fk = kk;
        frt = rt;
      }
    }
    const int s = k % ST;
    mbar_wait_opt(full0 + 8 * s, (uint32_t)(k / ST) & 1u, a.sleep);
    uint4 raw[8];
    const uint8_t* sp = smp + s * STAGE + off;
#pragma unroll
    for (int i = 0; i < 8; ++i) raw[i] = *reinterpret_cast<const uint4*>(sp + i * 16 * 128);
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * s);
    uint32_t cm[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t a0 = raw[i].x & 0x7FFF7FFFu, a1 = raw[i].y & 0x7FFF7FFFu;
      const uint32_t a2 = raw[i].z & 0x7FFF7FFFu, a3 = raw[i].w & 0x7FFF7FFFu;
      if (MODE & 4) {
        cm[0] = __vmaxu2(cm[0], a0); cm[1] = __vmaxu2(cm[1], a1);
        cm[2] = __vmaxu2(cm[2], a2); cm[3] = __vmaxu2(cm[3], a3);
      }
      if (MODE & 2) {
        const uint32_t m2 = __vmaxu2(__vmaxu2(a0, a1), __vmaxu2(a2, a3));
        rm[i] = max(rm[i], max(m2 & 0xFFFFu, m2 >> 16) << 16);
      }
    }
    if (MODE & 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        cm[j] = __vmaxu2(cm[j], __shfl_xor_sync(0xffffffffu, cm[j], 1));
        cm[j] = __vmaxu2(cm[j], __shfl_xor_sync(0xffffffffu, cm[j], 2));
        cm[j] = __vmaxu2(cm[j], __shfl_xor_sync(0xffffffffu, cm[j], 4));
        cm[j] = __vmaxu2(cm[j], __shfl_xor_sync(0xffffffffu, cm[j], 8));
      }
      if (r16 < 8) {   // lane r16 of each half-warp: column colw + r16 (word r16 / 2, high half if odd)
        const int j = r16 >> 1;
        const uint32_t w = j == 0 ? cm[0] : j == 1 ? cm[1] : j == 2 ? cm[2] : cm[3];
        const uint32_t v = (r16 & 1) ? (w & 0xFFFF0000u) : (w << 16);
        int64_t cbase = 0;
        if (kk == 0 && (a.seg.offs || a.seg.seg_rows > 0)) {
          int64_t sstart;
          cbase = (int64_t)seg_of(a.seg, (int64_t)rt * 128, sstart) * a.C[0];
        }
        if (v) atomicMax(a.col[kk] + cbase + (int64_t)ct * 128 + colw + r16, v);
      }
    }
  }
  if ((MODE & 2) && strip >= 0) flush_rows();
}

// Tensorwise amax of a contiguous tensor: persistent grid-stride stream of 16-byte vectors,
// 8 independent loads in flight per thread, |x| max on raw bit patterns (bf16: two 16-bit
// lanes per word via __vmaxu2), one atomicMax per CTA.
template <typename T, int U>
__global__ void __launch_bounds__(256) amax_flat_kernel(const uint4* __restrict__ x0, int64_t n0, uint32_t* out0,
                                                        const uint4* __restrict__ x1, int64_t n1, uint32_t* out1,
                                                        int g0) {
  // Each warp streams contiguous 512*U-byte chunks (U coalesced 512-B loads in flight per thread),
  // chunks strided over the grid; |x| max on raw bit patterns (bf16: two 16-bit lanes per word
  // via __vmaxu2), one atomicMax per CTA.  Two tensors (X and W of the forward): CTAs [0, g0) stream
  // the first, [g0, grid) the second.
  __shared__ uint32_t wred[8];
  const bool second = (int)blockIdx.x >= g0;
  const uint4* __restrict__ x = second ? x1 : x0;
  const int64_t n16 = second ? n1 : n0;
  uint32_t* out = second ? out1 : out0;
  const int64_t bid = second ? (int64_t)blockIdx.x - g0 : (int64_t)blockIdx.x;
  const int64_t nblk = second ? (int64_t)gridDim.x - g0 : (int64_t)g0;
  constexpr bool BF = sizeof(T) == 2;
  const uint32_t mask = BF ? 0x7FFF7FFFu : 0x7FFFFFFFu;
  uint32_t m = 0;
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (bid * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (nblk * blockDim.x) >> 5;
  auto fold = [&](const uint4& v) {
    if (BF) {
      m = __vmaxu2(m, v.x & mask); m = __vmaxu2(m, v.y & mask);
      m = __vmaxu2(m, v.z & mask); m = __vmaxu2(m, v.w & mask);
    } else {
      m = max(m, v.x & mask); m = max(m, v.y & mask); m = max(m, v.z & mask); m = max(m, v.w & mask);
    }
  };
  const int64_t nchunks = n16 / (32 * U);
  for (int64_t c = gwarp; c < nchunks; c += nwarps) {
    const uint4* p = x + c * (32 * U) + lane;
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(p + 32 * u);
#pragma unroll
    for (int u = 0; u < U; ++u) fold(v[u]);
  }
  for (int64_t i = nchunks * (32 * U) + gwarp * 32 + lane; i < n16; i += nwarps * 32) fold(__ldg(x + i));
  if (BF) m = max(m & 0xFFFFu, m >> 16) << 16;   // bf16 |x| bits -> fp32 bit pattern
  m = __reduce_max_sync(0xffffffffu, m);
  if (lane == 0) wred[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t r = wred[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = max(r, wred[w]);
    atomicMax(out, r);
  }
}

// Tensorwise amax of up to AMAX_MULTI_MAX tensors in one launch (the weights after an optimizer
// step: one pass instead of one launch per weight).  Work unit = a warp chunk of 32*8 16-byte
// vectors inside one row; the chunks of all tensors are numbered consecutively and every warp
// takes one contiguous range of them, so a warp crosses at most a few tensor boundaries and
// issues one atomicMax per (warp, tensor) it touched.
__global__ void __launch_bounds__(256) amax_multi_kernel(const __grid_constant__ AmaxMultiArgs a) {
  constexpr int U = 8;
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t total = a.chunk_start[a.n];
  const int64_t c_begin = total * gwarp / nwarps, c_end = total * (gwarp + 1) / nwarps;
  int t = 0;
  while (t + 1 < a.n && a.chunk_start[t + 1] <= c_begin) ++t;
  uint32_t m = 0;
  auto flush = [&](int tt) {
    const uint32_t r = __reduce_max_sync(0xffffffffu, m);
    if (lane == 0 && r) atomicMax(a.out + tt, r);
    m = 0;
  };
  for (int64_t c = c_begin; c < c_end; ++c) {
    if (c >= a.chunk_start[t + 1]) {   // warp-uniform
      flush(t);
      do { ++t; } while (c >= a.chunk_start[t + 1]);
    }
    const int64_t local = c - a.chunk_start[t];
    const int64_t row = local / a.cpr[t], seg = local - row * a.cpr[t];
    const uint4* p = reinterpret_cast<const uint4*>(a.ptr[t] + row * a.ld_bytes[t]) + seg * (32 * U);
    const int64_t rem = a.vecs[t] - seg * (32 * U);
    const int valid = rem < 32 * U ? (int)rem : 32 * U;
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = (lane + 32 * u < valid) ? __ldg(p + lane + 32 * u) : make_uint4(0, 0, 0, 0);
    if (a.bf16[t]) {
      uint32_t h = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        h = __vmaxu2(h, v[u].x & 0x7FFF7FFFu); h = __vmaxu2(h, v[u].y & 0x7FFF7FFFu);
        h = __vmaxu2(h, v[u].z & 0x7FFF7FFFu); h = __vmaxu2(h, v[u].w & 0x7FFF7FFFu);
      }
      m = max(m, max(h & 0xFFFFu, h >> 16) << 16);   // bf16 |x| bits -> fp32 bit pattern
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        m = max(m, v[u].x & 0x7FFFFFFFu); m = max(m, v[u].y & 0x7FFFFFFFu);
        m = max(m, v[u].z & 0x7FFFFFFFu); m = max(m, v[u].w & 0x7FFFFFFFu);
      }
    }
  }
  if (c_begin < c_end) flush(t);
}

// ---------------------------------------------------------------------------
// cast_tile: q (row-major) with scale mode QM, q_t (transposed) with scale mode TM.
// Modes: 0 none, 1 tensor (amax[1]), 2 per row (amax[R]), 3 per column (amax[C]).
// Scale outputs are written by the tiles on the first tile row / column.
// ---------------------------------------------------------------------------
template <typename T, int FMT, int QM, int TM_>
__device__ __forceinline__ void cast_tile_body(const T* __restrict__ x, int64_t R, int64_t C, int64_t ld,
                                               const float* __restrict__ amax_q, const float* __restrict__ amax_t,
                                               uint8_t* __restrict__ q, uint8_t* __restrict__ qt, float* scale_q,
                                               float* scale_t, const Seg& seg, int bx, int by) {
  // TM_ >= 4: the second output is written row-major ([R,C], like q) with scale mode TM_ - 2,
  // i.e. the column-scaled copy the backward GEMMs read MN-major (no transpose).
  constexpr bool TRM = TM_ >= 4;
  constexpr int TM = TRM ? TM_ - 2 : TM_;
  __shared__ __align__(16) uint32_t tile[128 * 32];
  __shared__ float sq[128];
  __shared__ float st[128];
  const int t = threadIdx.x;
  const int64_t r0 = (int64_t)by * 128, c0 = (int64_t)bx * 128;
  const int vrows = imin128(R - r0), vcols = imin128(C - c0);

  // Per-tile scale vectors (and the scale outputs).  `u` is the filling thread's index: with per-row AND
  // per-column vectors the rows are filled by threads 0..127 and the columns by threads 128..255, in parallel.
  auto fill = [&](int mode, const float* amax, float* sv, float* out, int u) {
    if (u < 0) return;
    if (mode == 1) {
      if (u == 0) {
        const float s = scale_of<FMT>(amax[0]);
        sv[0] = s;
        if (out && bx == 0 && by == 0) out[0] = s;
      }
    } else if (mode == 2) {
      if (u < vrows) {
        const float s = scale_of<FMT>(amax[r0 + u]);
        sv[u] = s;
        if (out && bx == 0) out[r0 + u] = s;
      }
    } else if (mode == 3) {   // per column (per segment of rows in the grouped recipe)
      if (u < vcols) {
        int64_t sstart;
        const int64_t cbase = (int64_t)seg_of(seg, r0, sstart) * C;
        const float s = scale_of<FMT>(amax[cbase + c0 + u]);
        sv[u] = s;
        if (out && r0 == sstart) out[cbase + c0 + u] = s;
      }
    }
  };
  const int cc = (t & 15) * 8;
  const bool cvalid = cc < vcols;
  // row (t >> 4) of the tile; row (t >> 4) + 16 i is 16 i rows further (64-bit products formed once)
  // (32-bit row offsets: 7 x 16 rows x ld elements stays far below 2^32 for any tensor the library accepts)
  const T* xrow = x + (r0 + (t >> 4)) * ld + c0 + cc;
  const uint32_t xstep = 16u * (uint32_t)ld;
  Raw8<T> raw[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int rr = (t >> 4) + 16 * i;
    if (cvalid && rr < vrows) raw[i].load(xrow + (uint32_t)i * xstep);
  }
  const int64_t orow = (r0 + (t >> 4)) * C + c0 + cc;
  const uint32_t ostep = 16u * (uint32_t)C;
  constexpr bool split = QM >= 2 && TM >= 2 && QM != TM;   // a row and a column vector: one half of the CTA each
  if (split) {
    if (t < 128) fill(QM, amax_q, sq, scale_q, t);
    else fill(TM, amax_t, st, scale_t, t - 128);
  } else {
    fill(QM, amax_q, sq, scale_q, t);
    fill(TM, amax_t, st, scale_t, t);
  }
  __syncthreads();

#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int rr = (t >> 4) + 16 * i;
    if (!cvalid || rr >= vrows) continue;
    float v[8];
    raw[i].get(v);
    uint2 bq = make_uint2(0, 0), bt = make_uint2(0, 0);
    if (QM != 0) {
      if (QM == 1) bq = cast8<FMT>(v, sq[0]);
      if (QM == 2) bq = cast8<FMT>(v, sq[rr]);
      if (QM == 3) bq = cast8v<FMT>(v, &sq[cc]);
      *reinterpret_cast<uint2*>(q + orow + (uint32_t)i * ostep) = bq;
    }
    if (TM != 0) {
      if (TM == QM) bt = bq;
      else if (TM == 1) bt = cast8<FMT>(v, st[0]);
      else if (TM == 2) bt = cast8<FMT>(v, st[rr]);
      else bt = cast8v<FMT>(v, &st[cc]);
      if (TRM) *reinterpret_cast<uint2*>(qt + orow + (uint32_t)i * ostep) = bt;
      else *reinterpret_cast<uint2*>(&tile[swz(rr, cc >> 2)]) = bt;
    }
  }
  if (TM != 0 && !TRM) {
    __syncthreads();
    store_transposed(tile, qt, R, r0, c0, vrows, vcols);
  }
}

template <typename T, int FMT, int QM, int TM_>
__global__ void __launch_bounds__(256) cast_tile_kernel(const T* __restrict__ x, int64_t R, int64_t C, int64_t ld,
                                                        const float* __restrict__ amax_q,
                                                        const float* __restrict__ amax_t, uint8_t* __restrict__ q,
                                                        uint8_t* __restrict__ qt, float* scale_q, float* scale_t,
                                                        const Seg seg) {
  // tiles in decreasing linear order: the first tiles read are the ones amax_tile read last
  const int rtile = (int)(gridDim.x * gridDim.y - 1 - (blockIdx.y * gridDim.x + blockIdx.x));
  cast_tile_body<T, FMT, QM, TM_>(x, R, C, ld, amax_q, amax_t, q, qt, scale_q, scale_t, seg,
                                  rtile % (int)gridDim.x, rtile / (int)gridDim.x);
}

// Several tensors (the forward's X and W; a shared-input group's X and every W_i, or every member's dY)
// cast by one launch: a 1-D grid over the tiles of all, walked in decreasing order over
// [tensor 0 tiles, tensor 1 tiles, ...] (the reverse of the multi-tensor amax launch), so the small
// tensors cost no launch ramp and tail of their own.
template <typename T, int FMT, int QM, int TM_>
__global__ void __launch_bounds__(256) cast_tile_dual_kernel(const __grid_constant__ CastMulti a) {
  int id = a.tstart[a.n] - 1 - (int)blockIdx.x;
  int k = 0;
  while (k + 1 < a.n && id >= a.tstart[k + 1]) ++k;
  id -= a.tstart[k];
  const int tx = (int)((a.C[k] + 127) / 128);
  cast_tile_body<T, FMT, QM, TM_>(static_cast<const T*>(a.x[k]), a.R[k], a.C[k], a.ld[k], a.amax_q[k], a.amax_t[k],
                                  a.q[k], a.qt[k], a.scale_q[k], a.scale_t[k], Seg{}, id % tx, id / tx);
}

// ---------------------------------------------------------------------------
// Rowwise casts, persistent TMA variant (bf16, rows and columns multiples of 128; knob cast_rc_tma): the
// same arithmetic and bytes as cast_tile_kernel<bf16, FMT, 2, 5> (row-scaled codes q and column-scaled codes
// qt, both row-major), for up to CAST_MULTI_MAX tensors per launch.  CTA b walks tiles total-1-b,
// total-1-b-G, ... (the reverse of the amax launch's order, so the first reads find the amax's last tiles
// in L2); thread 0 streams the bf16 tiles into a 3-deep ring; per tile the 128 row and 128 column scales
// are computed into smem, every thread casts 8 rows x 8 columns twice, writes both code tiles into the
// tile's own ring stage, and thread 0 sends them out by two TMA tensor stores (the stage is refilled one
// tile later, after the stores have read it).
// ---------------------------------------------------------------------------
template <int FMT, int ST, int NT>   // NT threads: 256 (2 CTAs per SM) or 512 (1 CTA per SM, deeper ring)
__global__ void __launch_bounds__(NT, 1) cast_rc_tma_kernel(const __grid_constant__ CastRCArgs a) {
  constexpr int RPT = 2048 / NT;   // rows per thread (8 columns each)
  constexpr int STAGE = 128 * 256;
  extern __shared__ __align__(1024) uint8_t sm[];
  float* srow = reinterpret_cast<float*>(sm + ST * STAGE);
  float* scol = srow + 128;
  const uint32_t stage0 = smem_u32(sm), bar0 = smem_u32(sm + ST * STAGE + 1024);
  const int t = threadIdx.x;
  const int total = a.tstart[a.n];
  const int G = (int)gridDim.x;
  auto where = [&](int id, int& k, int& rt, int& ct) {
    k = 0;
    while (k + 1 < a.n && id >= a.tstart[k + 1]) ++k;
    const int local = id - a.tstart[k];
    rt = local / a.tiles_x[k];
    ct = local - rt * a.tiles_x[k];
  };
  auto issue = [&](int k) {   // thread 0: the k-th tile of this CTA into stage k % ST
    const int j = (int)blockIdx.x + k * G;
    if (j < total) {
      int kk, rt, ct;
      where(total - 1 - j, kk, rt, ct);
      const uint32_t bar = bar0 + 8 * (k % ST);
      mbar_arrive_expect_tx(bar, STAGE);
      tma_load_2d(stage0 + (k % ST) * STAGE, &a.in[kk], ct * 128, rt * 128, bar, l2_policy_evict_first());
    }
  };
  if (t == 0) {
    for (int i = 0; i < a.n; ++i) tma_prefetch_desc(&a.in[i]);
    for (int i = 0; i < ST; ++i) mbar_init(bar0 + 8 * i, 1);
    fence_mbar_init();
    for (int k = 0; k < ST; ++k) issue(k);
  }
  __syncthreads();
  const int cc = (t & 15) * 8, rbase = RPT * (t >> 4);
  for (int k = 0;; ++k) {
    const int j = (int)blockIdx.x + k * G;
    if (j >= total) break;
    int kk, rt, ct;
    where(total - 1 - j, kk, rt, ct);
    const int64_t r0 = (int64_t)rt * 128, c0 = (int64_t)ct * 128;
    const int s = k % ST;
    // this tile's scales (row t for t < 128, column t - 128 otherwise); the scale outputs are written by the
    // tiles of the first tile column (rows) / first tile row (columns), as cast_tile_kernel does
    if (t < 128) {
      const float sc = scale_of<FMT>(a.amax_q[kk][r0 + t]);
      srow[t] = sc;
      if (ct == 0 && a.scale_q[kk]) a.scale_q[kk][r0 + t] = sc;
    } else if (t < 256) {
      const float sc = scale_of<FMT>(a.amax_t[kk][c0 + t - 128]);
      scol[t - 128] = sc;
      if (rt == 0 && a.scale_t[kk]) a.scale_t[kk][c0 + t - 128] = sc;
    }
    mbar_wait(bar0 + 8 * s, (uint32_t)(k / ST) & 1u);
    uint4 raw[RPT];
    const uint8_t* sp = sm + s * STAGE + rbase * 256 + cc * 2;
#pragma unroll
    for (int i = 0; i < RPT; ++i) raw[i] = *reinterpret_cast<const uint4*>(sp + i * 256);
    __syncthreads();                       // (1) stage read by every thread, scales visible
    if (t == 0) {
      fence_proxy_async_smem();
      if (k > 0) {   // tile k-1's code stores were issued from its stage: refill it once they have read it
        bulk_wait_read0();
        issue(k - 1 + ST);
      }
    }
    float sv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) sv[q] = scol[cc + q];
    uint8_t* dst = sm + s * STAGE;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      float v[8];
      const uint32_t w[4] = {raw[i].x, raw[i].y, raw[i].z, raw[i].w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        v[2 * q] = __uint_as_float(w[q] << 16);
        v[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
      }
      *reinterpret_cast<uint2*>(dst + (rbase + i) * 128 + cc) = cast8<FMT>(v, srow[rbase + i]);
      *reinterpret_cast<uint2*>(dst + 16384 + (rbase + i) * 128 + cc) = cast8v<FMT>(v, sv);
    }
    fence_proxy_async_smem();
    __syncthreads();                       // (2) both code tiles written; scales free for the next tile
    if (t == 0) {
      tma_store_2d(&a.oq[kk], stage0 + s * STAGE, (int)c0, (int)r0);
      tma_store_2d(&a.ot[kk], stage0 + s * STAGE + 16384, (int)c0, (int)r0);
      bulk_commit_group();
    }
  }
  if (t == 0) bulk_wait_all0();
}

// ---------------------------------------------------------------------------
// MXFP8 cast, dim0 (blocks of 32 along columns, row-major out) and dim1 (blocks
// of 32 along rows, transposed out) from one read of a 128 x 128 tile.
// E8M0 codes by integer exponent arithmetic (R-c12):
//   FLOOR: c = clamp(E - emax, 0, 254)              E = fp32 exponent field of amax
//   RCEIL: c = clamp(E - emax + (mant > 0x600000), 0, 254), E == 0 -> 0
// (mant > 0x600000  <=>  amax mantissa > 1.75 = fmax mantissa)
// Elements: satRNE(RN32(x * 2^(127-c))), no flush-to-zero (R-c11).
// Scales are written in the blocked 128x4 layout of fp8train.h.
// ---------------------------------------------------------------------------
template <int FMT, bool RCEIL>
__device__ __forceinline__ uint32_t e8m0_code(uint32_t amax_bits) {
  // E == 0 (zero or subnormal amax) needs no branch: E - emax (+ 1) < 0 clamps to code 0
  const int E = (int)(amax_bits >> 23);
  int c = E - kEmax<FMT>();
  if (RCEIL && (amax_bits & 0x7FFFFFu) > 0x600000u) c += 1;
  return (uint32_t)min(max(c, 0), 254);
}
// 2^(127 - c) as fp32 (c = 254 -> 2^-127, a subnormal).
__device__ __forceinline__ float e8m0_mult(uint32_t c) {
  return c < 254 ? __uint_as_float((254u - c) << 23) : __uint_as_float(0x00400000u);
}
__device__ __forceinline__ int64_t sf_offset(int64_t r, int64_t cblk, int64_t ncol_tiles) {
  // logical (row r, 32-block column cblk) of a [R, C/32] code matrix, 128x4 tiles
  return ((r >> 7) * ncol_tiles + (cblk >> 2)) * 512 + (r & 31) * 16 + ((r >> 5) & 3) * 4 + (cblk & 3);
}

template <typename T, int FMT, bool RCEIL, bool DIM0, bool DIM1, bool TR1>
__global__ void __launch_bounds__(256, 3) mx_cast_kernel(const T* __restrict__ x, int64_t R, int64_t C, int64_t ld,
                                                      uint8_t* __restrict__ q0, uint8_t* __restrict__ sf0,
                                                      uint8_t* __restrict__ q1, uint8_t* __restrict__ sf1) {
  // Thread t owns 8 consecutive rows (8*(t/16) .. +7) x 8 consecutive columns (8*(t%16) .. +7)
  // of the 128 x 128 tile.  dim0 blocks (32 columns of one row) span 4 lanes; dim1 blocks
  // (32 rows of one column) span the two half-warps of warps 2j and 2j+1.
  __shared__ __align__(16) uint32_t tile[128 * 32];
  __shared__ __align__(16) uint32_t red[8][128];
  __shared__ __align__(16) float mult1[4][128];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t r0 = (int64_t)blockIdx.y * 128, c0 = (int64_t)blockIdx.x * 128;
  const int cc = (t & 15) * 8;
  const int rbase = 8 * (t >> 4);
  Raw8<T> raw[8];
  const T* xp = x + (r0 + rbase) * ld + c0 + cc;
#pragma unroll
  for (int i = 0; i < 8; ++i) raw[i].load(xp + i * ld);

  // one pass over the 8 rows: dim0 block codes + casts, and the dim1 column maxima
  uint32_t cm[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint8_t* q0p = DIM0 ? q0 + (r0 + rbase) * C + c0 + cc : nullptr;
  // E8M0 blocked offset of (row r0+rbase+i, 32-block (c0+cc)/32): rows of a 128-row tile are
  // 16 B apart within each group of 32 and 4 B apart across groups
  const int64_t sf0_base = (((r0 >> 7) * (C >> 7) + (c0 >> 7)) * 512) + ((rbase >> 5) & 3) * 4 + (cc >> 5);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float v[8];
    raw[i].get(v);
    uint32_t m = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t a = abs_bits(v[e]);
      m = max(m, a);
      if (DIM1) cm[e] = max(cm[e], a);
    }
    if (DIM0) {
      m = max(m, __shfl_xor_sync(0xffffffffu, m, 1));
      m = max(m, __shfl_xor_sync(0xffffffffu, m, 2));
      const uint32_t code = e8m0_code<FMT, RCEIL>(m);
      *reinterpret_cast<uint2*>(q0p + i * C) = cast8<FMT>(v, e8m0_mult(code));
      if ((t & 3) == 0) sf0[sf0_base + ((rbase + i) & 31) * 16] = (uint8_t)code;
    }
  }
  if (DIM1) {
#pragma unroll
    for (int e = 0; e < 8; ++e) cm[e] = max(cm[e], __shfl_xor_sync(0xffffffffu, cm[e], 16));
    if (lane < 16) {
      *reinterpret_cast<uint4*>(&red[warp][cc]) = make_uint4(cm[0], cm[1], cm[2], cm[3]);
      *reinterpret_cast<uint4*>(&red[warp][cc + 4]) = make_uint4(cm[4], cm[5], cm[6], cm[7]);
    }
    __syncthreads();
    {
      const int j = t >> 6, col = (t & 63) * 2;   // 32-row block j, columns col, col+1
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t m = max(red[2 * j][col + h], red[2 * j + 1][col + h]);
        const uint32_t code = e8m0_code<FMT, RCEIL>(m);
        mult1[j][col + h] = e8m0_mult(code);
        sf1[sf_offset(c0 + col + h, (r0 >> 5) + j, R >> 7)] = (uint8_t)code;
      }
    }
    __syncthreads();
    const int j = t >> 6;                          // all 8 rows of this thread lie in block j
    const float4 ma = *reinterpret_cast<const float4*>(&mult1[j][cc]);
    const float4 mb = *reinterpret_cast<const float4*>(&mult1[j][cc + 4]);
    const float mu[8] = {ma.x, ma.y, ma.z, ma.w, mb.x, mb.y, mb.z, mb.w};
    if (TR1) {   // q1 = the dim1 codes transposed, [C, R] (K-major for the backward GEMMs)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float v[8];
        raw[i].get(v);
        *reinterpret_cast<uint2*>(&tile[swz(rbase + i, cc >> 2)]) = cast8v<FMT>(v, mu);
      }
      __syncthreads();
      store_transposed(tile, q1, R, r0, c0, 128, 128);
    } else {     // q1 = the dim1 codes in the input's layout, [R, C] (read MN-major by the GEMMs)
      uint8_t* q1p = q1 + (r0 + rbase) * C + c0 + cc;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float v[8];
        raw[i].get(v);
        *reinterpret_cast<uint2*>(q1p + i * C) = cast8v<FMT>(v, mu);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// MXFP8 cast, TMA-pipelined persistent variant (bf16 input; rows, cols multiples of 128).
// Same arithmetic and outputs as mx_cast_kernel.  CTA b walks tiles b, b+G, b+2G, ...;
// thread 0 streams the 128 x 128 bf16 tiles (32 KB) into an ST-deep shared-memory ring with
// cp.async.bulk.tensor, so the HBM reads of the next ST tiles stay in flight while the 8 warps
// reduce and cast the current one.  |x| maxima run on packed bf16 pairs (__vmaxu2 on the raw
// bits), the power-of-two scaling on fp32 pairs (__fmul2_rn, IEEE RN, no FTZ), and each
// tile's two 512-byte E8M0 scale tiles leave as 16-byte stores.
// ---------------------------------------------------------------------------
template <int ST, bool TR1> struct MxSmem {
  static constexpr int STAGE = 128 * 256;             // one bf16 tile, row-major, 256 B per row
  static constexpr int RED = ST * STAGE;              // u32 [8][64]: per-warp packed column maxima
  static constexpr int MULT = RED + 8 * 64 * 4;       // f32 [4][128]: dim1 multipliers
  static constexpr int SF0 = MULT + 4 * 128 * 4;      // u8 [512]: dim0 E8M0 tile (blocked layout)
  static constexpr int SF1 = SF0 + 512;               // u8 [512]: dim1 E8M0 tile
  static constexpr int TILE = SF1 + 512;              // u32 [128*32]: transposed staging (TR1)
  static constexpr int BAR = TILE + (TR1 ? 128 * 32 * 4 : 0);
  static constexpr int BYTES = BAR + ST * 8;
};

// 8 bf16 (4 packed words) -> 8 FP8 codes of x * mult (pairs of fp32 multipliers m[0..3]).
template <int FMT>
__device__ __forceinline__ uint2 cast8_bf16x2(const uint32_t (&w)[4], const float2 (&m)[4]) {
  uint32_t b[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 p = __fmul2_rn(make_float2(__uint_as_float(w[j] << 16), __uint_as_float(w[j] & 0xFFFF0000u)), m[j]);
    b[j] = FMT == 0 ? cvt_e4m3x2(p.y, p.x) : cvt_e5m2x2(p.y, p.x);
  }
  return make_uint2(b[0] | (b[1] << 16), b[2] | (b[3] << 16));
}

// 8 fp32 values (pairs) -> 8 FP8 codes of x * mult.
template <int FMT>
__device__ __forceinline__ uint2 cast8_f32x2(const float2 (&f)[4], const float2 (&m)[4]) {
  uint32_t b[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 p = __fmul2_rn(f[q], m[q]);
    b[q] = FMT == 0 ? cvt_e4m3x2(p.y, p.x) : cvt_e5m2x2(p.y, p.x);
  }
  return make_uint2(b[0] | (b[1] << 16), b[2] | (b[3] << 16));
}

// TS (knob mx_cast_tstore; dim0 + row-major dim1 only): the codes are written into the tile's own ring stage
// (its bf16 data is in registers by then) and leave as two 16 KB TMA tensor stores; the stage is refilled
// one tile later, once the stores have read it.
template <int FMT, bool RCEIL, bool DIM0, bool DIM1, bool TR1, int ST, bool TS = false>
// ST == 2 (knob mx_cast_occ3): a 2-deep ring and <= 85 registers, so 3 CTAs (24 warps) share an SM
__global__ void __launch_bounds__(256, (ST == 2 && !TR1) ? 3 : 1) mx_cast_tma_kernel(const __grid_constant__ CUtensorMap tmap, int64_t R,
                                                          int64_t C, uint8_t* __restrict__ q0,
                                                          uint8_t* __restrict__ sf0, uint8_t* __restrict__ q1,
                                                          uint8_t* __restrict__ sf1, int dbg,
                                                          const __grid_constant__ CUtensorMap tq0,
                                                          const __grid_constant__ CUtensorMap tq1) {
  static_assert(!TS || (DIM0 && DIM1 && !TR1), "TMA-store variant: dim0 + row-major dim1 only");
  using L = MxSmem<ST, TR1>;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint32_t(*red)[64] = reinterpret_cast<uint32_t(*)[64]>(sm + L::RED);
  float(*mult1)[128] = reinterpret_cast<float(*)[128]>(sm + L::MULT);
  uint8_t* s_sf0 = sm + L::SF0;
  uint8_t* s_sf1 = sm + L::SF1;
  uint32_t* tile = reinterpret_cast<uint32_t*>(sm + L::TILE);
  const uint32_t bar0 = smem_u32(sm + L::BAR), stage0 = smem_u32(sm);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int tiles_x = (int)(C >> 7);
  const int num_tiles = tiles_x * (int)(R >> 7);
  const int G = (int)gridDim.x;
  auto issue = [&](int k) {   // thread 0: TMA of this CTA's k-th tile into stage k % ST
    const int id = (int)blockIdx.x + k * G;
    if (id < num_tiles) {
      const uint32_t bar = bar0 + 8 * (k % ST);
      mbar_arrive_expect_tx(bar, L::STAGE);
      tma_load_2d(stage0 + (k % ST) * L::STAGE, &tmap, (id % tiles_x) * 128, (id / tiles_x) * 128, bar,
                  l2_policy_evict_first());
    }
  };
  if (t == 0) {
    tma_prefetch_desc(&tmap);
    for (int i = 0; i < ST; ++i) mbar_init(bar0 + 8 * i, 1);
    fence_mbar_init();
    for (int k = 0; k < ST; ++k) issue(k);
  }
  __syncthreads();
  const int cc = (t & 15) * 8, rbase = 8 * (t >> 4);
  // tiles b, b + G, b + 2G, ...: (row, column) tile by a cursor -- G = gq * tiles_x + gr, one compare per step
  const int gq = G / tiles_x, gr = G - gq * tiles_x;
  int trow = (int)blockIdx.x / tiles_x, tcol = (int)blockIdx.x - trow * tiles_x;
  for (int k = 0;; ++k, trow += gq, tcol += gr) {
    if (tcol >= tiles_x) {
      tcol -= tiles_x;
      ++trow;
    }
    const int id = (int)blockIdx.x + k * G;
    if (id >= num_tiles) break;
    const int64_t r0 = (int64_t)trow * 128, c0 = (int64_t)tcol * 128;
    mbar_wait(bar0 + 8 * (k % ST), (uint32_t)(k / ST) & 1u);
    uint4 raw[8];
    const uint8_t* sp = sm + (k % ST) * L::STAGE + rbase * 256 + cc * 2;
#pragma unroll
    for (int i = 0; i < 8; ++i) raw[i] = *reinterpret_cast<const uint4*>(sp + i * 256);
    if (!TS) {   // TS: the stage is overwritten by this tile's codes only after barrier (2), which every thread
                 // reaches after its loads above -- no barrier of its own
      __syncthreads();                     // (1) stage consumed by every thread
      if (t == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(k + ST);
      }
    }

    // pass 1 over the raw words: packed |x| maxima per row (dim0, this thread's 8 columns) and per column
    // (dim1, this thread's 8 rows)
    uint32_t cmw[4] = {0, 0, 0, 0};
    uint32_t rmx[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t a0 = raw[i].x & 0x7FFF7FFFu, a1 = raw[i].y & 0x7FFF7FFFu;
      const uint32_t a2 = raw[i].z & 0x7FFF7FFFu, a3 = raw[i].w & 0x7FFF7FFFu;
      if (DIM1) {
        cmw[0] = __vmaxu2(cmw[0], a0); cmw[1] = __vmaxu2(cmw[1], a1);
        cmw[2] = __vmaxu2(cmw[2], a2); cmw[3] = __vmaxu2(cmw[3], a3);
      }
      if (DIM0) rmx[i] = __vmaxu2(__vmaxu2(a0, a1), __vmaxu2(a2, a3));
    }
    // dim0 block codes (4 lanes per 32-column block; all 4 store the same byte)
    float mu0[8];
    if (DIM0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint32_t m = max(rmx[i] & 0xFFFFu, rmx[i] >> 16);
        m = max(m, __shfl_xor_sync(0xffffffffu, m, 1));
        m = max(m, __shfl_xor_sync(0xffffffffu, m, 2));
        const uint32_t code = e8m0_code<FMT, RCEIL>(m << 16);
        mu0[i] = e8m0_mult(code);
        const int rr = rbase + i;
        s_sf0[(rr & 31) * 16 + (rr >> 5) * 4 + (cc >> 5)] = (uint8_t)code;
      }
    }
    const int64_t base0 = ((r0 >> 7) * (C >> 7) + (c0 >> 7)) * 512;
    float2 mu[4];
    if (DIM1) {
#pragma unroll
      for (int j = 0; j < 4; ++j) cmw[j] = __vmaxu2(cmw[j], __shfl_xor_sync(0xffffffffu, cmw[j], 16));
      if (lane < 16) *reinterpret_cast<uint4*>(&red[warp][cc >> 1]) = make_uint4(cmw[0], cmw[1], cmw[2], cmw[3]);
      __syncthreads();                     // (2)
      if (TS && t == 0 && k > 0) {   // tile k-1's code stores were issued from its stage: refill it once read
        bulk_wait_read0();
        fence_proxy_async_smem();
        issue(k - 1 + ST);
      }
      {
        const int j = t >> 6, wp = t & 63;   // 32-row block j, columns 2wp, 2wp+1
        const uint32_t m2 = __vmaxu2(red[2 * j][wp], red[2 * j + 1][wp]);
        const uint32_t clo = e8m0_code<FMT, RCEIL>(m2 << 16), chi = e8m0_code<FMT, RCEIL>(m2 & 0xFFFF0000u);
        *reinterpret_cast<float2*>(&mult1[j][2 * wp]) = make_float2(e8m0_mult(clo), e8m0_mult(chi));
        const int c = 2 * wp;
        s_sf1[(c & 31) * 16 + (c >> 5) * 4 + j] = (uint8_t)clo;
        s_sf1[((c + 1) & 31) * 16 + ((c + 1) >> 5) * 4 + j] = (uint8_t)chi;
      }
      __syncthreads();                     // (3)
      if (DIM0 && t < 32)
        *reinterpret_cast<uint4*>(sf0 + base0 + t * 16) = *reinterpret_cast<const uint4*>(s_sf0 + t * 16);
      if (t >= 32 && t < 64)
        *reinterpret_cast<uint4*>(sf1 + ((c0 >> 7) * (R >> 7) + (r0 >> 7)) * 512 + (t - 32) * 16) =
            *reinterpret_cast<const uint4*>(s_sf1 + (t - 32) * 16);
      const int j = t >> 6;                // all 8 rows of this thread lie in 32-row block j
      const float4 ma = *reinterpret_cast<const float4*>(&mult1[j][cc]);
      const float4 mb = *reinterpret_cast<const float4*>(&mult1[j][cc + 4]);
      mu[0] = make_float2(ma.x, ma.y); mu[1] = make_float2(ma.z, ma.w);
      mu[2] = make_float2(mb.x, mb.y); mu[3] = make_float2(mb.z, mb.w);
    }
    // pass 2: each row unpacked once and cast with both multipliers
    uint8_t* o0 = DIM0 ? q0 + (r0 + rbase) * C + c0 + cc : nullptr;
    uint8_t* o1 = DIM1 && !TR1 ? q1 + (r0 + rbase) * C + c0 + cc : nullptr;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float2 f[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t w = q == 0 ? raw[i].x : q == 1 ? raw[i].y : q == 2 ? raw[i].z : raw[i].w;
        f[q] = make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
      }
      if (DIM0) {
        const float2 mm[4] = {make_float2(mu0[i], mu0[i]), make_float2(mu0[i], mu0[i]), make_float2(mu0[i], mu0[i]),
                              make_float2(mu0[i], mu0[i])};
        const uint2 b0 = cast8_f32x2<FMT>(f, mm);
        if (TS) *reinterpret_cast<uint2*>(sm + (k % ST) * L::STAGE + (rbase + i) * 128 + cc) = b0;
        else if (!(dbg & 1)) *reinterpret_cast<uint2*>(o0 + i * C) = b0;
        else if (b0.x == 0x12345678u) q0[0] = 0;   // A/B probe (no stores): keep the cast alive
      }
      if (DIM1) {
        const uint2 b = cast8_f32x2<FMT>(f, mu);
        if (TR1) *reinterpret_cast<uint2*>(&tile[swz(rbase + i, cc >> 2)]) = b;
        else if (TS) *reinterpret_cast<uint2*>(sm + (k % ST) * L::STAGE + 16384 + (rbase + i) * 128 + cc) = b;
        else if (!(dbg & 1)) *reinterpret_cast<uint2*>(o1 + i * C) = b;
        else if (b.x == 0x12345678u) q1[0] = 0;
      }
    }
    if (TS) {   // both 128 x 128 code tiles of this tile -> global by TMA
      fence_proxy_async_smem();
      __syncthreads();                     // (4)
      if (t == 0) {
        const uint32_t st_s = stage0 + (k % ST) * L::STAGE;
        tma_store_2d(&tq0, st_s, (int)c0, (int)r0);
        tma_store_2d(&tq1, st_s + 16384, (int)c0, (int)r0);
        bulk_commit_group();
      }
    }
    if (DIM1) {
      if (TR1) {
        __syncthreads();                   // (4)
        store_transposed(tile, q1, R, r0, c0, 128, 128);
      }
    } else {
      __syncthreads();
      if (t < 32) *reinterpret_cast<uint4*>(sf0 + base0 + t * 16) = *reinterpret_cast<const uint4*>(s_sf0 + t * 16);
    }
  }
  if (TS && t == 0) bulk_wait_all0();   // the stores have read shared memory and completed before the CTA exits
}

// ---------------------------------------------------------------------------
// MXFP8 cast, warp-specialised variant (knob mx_cast_ws, the product path for bf16 inputs with row-major
// dim1 copies).  Same arithmetic and outputs as mx_cast_tma_kernel; what changes is who reduces what:
//   * warp 8 streams the 128 x 128 bf16 tiles (CTA b: tiles b, b + G, ...) into an ST-deep ring (full
//     barrier: TMA bytes; empty barrier: one arrival per consumer warp, right after its loads);
//   * consumer warp w owns one dim1 block -- rows [32 (w >> 1), +32) -- and 64 columns (w & 1): lane l
//     holds 8 columns (8 (l & 7)) of the 8 rows 8 (l >> 3) + i, so the dim1 column maxima of its block
//     are two xor shuffles (8, 16) away and no block-wide reduction is needed; dim0 blocks (32
//     columns) are 4 lanes, two xor shuffles (1, 2), as before;
//   * the tile's E8M0 codes are staged in a double-buffered 1 KB smem tile and leave as 16-byte stores
//     one tile later, after the one named barrier per tile among the consumer warps.
// ---------------------------------------------------------------------------
template <int FMT, bool RCEIL, bool DIM0, bool DIM1, int ST>
__global__ void __launch_bounds__(288, 2) mx_cast_ws_kernel(const __grid_constant__ CUtensorMap tmap, int64_t R,
                                                          int64_t C, uint8_t* __restrict__ q0,
                                                          uint8_t* __restrict__ sf0, uint8_t* __restrict__ q1,
                                                          uint8_t* __restrict__ sf1, int sleep) {
  constexpr int STAGE = 128 * 256;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sfb = sm + ST * STAGE;                       // [2][1024]: dim0 tile (512 B) + dim1 tile (512 B)
  const uint32_t stage0 = smem_u32(sm), full0 = smem_u32(sm + ST * STAGE + 2048), empty0 = full0 + 8 * ST;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int tiles_x = (int)(C >> 7);
  const int num_tiles = tiles_x * (int)(R >> 7);
  const int G = (int)gridDim.x;
  if (t == 0) {
    for (int i = 0; i < ST; ++i) {
      mbar_init(full0 + 8 * i, 1);
      mbar_init(empty0 + 8 * i, 8);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 8) {   // producer
    if (lane == 0) {
      tma_prefetch_desc(&tmap);
      const uint64_t pol = l2_policy_evict_first();
      for (int k = 0;; ++k) {
        const int id = (int)blockIdx.x + k * G;
        if (id >= num_tiles) break;
        const int s = k % ST;
        if (k >= ST) {
          mbar_wait_opt(empty0 + 8 * s, (uint32_t)(k / ST - 1) & 1u, sleep);
          fence_proxy_async_smem();
        }
        mbar_arrive_expect_tx(full0 + 8 * s, STAGE);
        tma_load_2d(stage0 + s * STAGE, &tmap, (id % tiles_x) * 128, (id / tiles_x) * 128, full0 + 8 * s, pol);
      }
    }
    return;
  }
  const int j = warp >> 1, h = warp & 1;                 // dim1 block (32 rows) and column half of this warp
  const int cl = 64 * h + 8 * (lane & 7);                // first of the lane's 8 columns
  const int rl = 32 * j + 8 * (lane >> 3);               // first of the lane's 8 rows
  // E8M0 positions in the blocked 512-byte tile: byte (r & 31) * 16 + (r >> 5) * 4 + (c >> 5)
  const int p0 = (8 * (lane >> 3)) * 16 + j * 4 + (cl >> 5);   // + 16 i for row rl + i (dim0)
  auto store_sf = [&](int buf, int64_t pr0, int64_t pc0) {     // threads 0..63: the previous tile's codes
    if (t < 64) {
      const uint4 v = *reinterpret_cast<const uint4*>(sfb + buf * 1024 + t * 16);
      if (t < 32) {
        if (DIM0) *reinterpret_cast<uint4*>(sf0 + ((pr0 >> 7) * (C >> 7) + (pc0 >> 7)) * 512 + t * 16) = v;
      } else if (DIM1) {
        *reinterpret_cast<uint4*>(sf1 + ((pc0 >> 7) * (R >> 7) + (pr0 >> 7)) * 512 + (t - 32) * 16) = v;
      }
    }
  };
  int64_t pr0 = 0, pc0 = 0;
  for (int k = 0;; ++k) {
    const int id = (int)blockIdx.x + k * G;
    if (id >= num_tiles) break;
    const int s = k % ST;
    const int64_t r0 = (int64_t)(id / tiles_x) * 128, c0 = (int64_t)(id % tiles_x) * 128;
    mbar_wait_opt(full0 + 8 * s, (uint32_t)(k / ST) & 1u, sleep);
    uint4 raw[8];
    const uint8_t* sp = sm + s * STAGE + rl * 256 + cl * 2;
#pragma unroll
    for (int i = 0; i < 8; ++i) raw[i] = *reinterpret_cast<const uint4*>(sp + i * 256);
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * s);
    // every consumer warp has finished tile k-1 (its codes are in sfb[(k-1) & 1]) and has stored the codes
    // of tile k-2 from sfb[k & 1]
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (k > 0) store_sf((k - 1) & 1, pr0, pc0);
    uint8_t* sb = sfb + (k & 1) * 1024;
    // pass 1 over the raw words: packed |x| maxima -- per row (dim0, over the lane's 8 columns) and per
    // column (dim1, over the lane's 8 rows)
    uint32_t rmx[8];
    uint32_t cm[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t a0 = raw[i].x & 0x7FFF7FFFu, a1 = raw[i].y & 0x7FFF7FFFu;
      const uint32_t a2 = raw[i].z & 0x7FFF7FFFu, a3 = raw[i].w & 0x7FFF7FFFu;
      if (DIM1) {
        cm[0] = __vmaxu2(cm[0], a0); cm[1] = __vmaxu2(cm[1], a1);
        cm[2] = __vmaxu2(cm[2], a2); cm[3] = __vmaxu2(cm[3], a3);
      }
      if (DIM0) rmx[i] = __vmaxu2(__vmaxu2(a0, a1), __vmaxu2(a2, a3));
    }
    // dim1 block codes (all lanes of a column hold the same maxima after the shuffles, so every lane stores
    // its codes: identical bytes to identical addresses, no divergent branch)
    float2 mu1[4];
    if (DIM1) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        cm[q] = __vmaxu2(cm[q], __shfl_xor_sync(0xffffffffu, cm[q], 8));
        cm[q] = __vmaxu2(cm[q], __shfl_xor_sync(0xffffffffu, cm[q], 16));
        const uint32_t clo = e8m0_code<FMT, RCEIL>(cm[q] << 16), chi = e8m0_code<FMT, RCEIL>(cm[q] & 0xFFFF0000u);
        mu1[q] = make_float2(e8m0_mult(clo), e8m0_mult(chi));
        const int c = cl + 2 * q;   // columns c, c + 1 of dim1 block j
        sb[512 + (c & 31) * 16 + (c >> 5) * 4 + j] = (uint8_t)clo;
        sb[512 + ((c + 1) & 31) * 16 + ((c + 1) >> 5) * 4 + j] = (uint8_t)chi;
      }
    }
    // dim0 block codes: 4 lanes per 32-column block (the 4 lanes store the same byte)
    float mu0[8];
    if (DIM0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint32_t m = max(rmx[i] & 0xFFFFu, rmx[i] >> 16);
        m = max(m, __shfl_xor_sync(0xffffffffu, m, 1));
        m = max(m, __shfl_xor_sync(0xffffffffu, m, 2));
        const uint32_t code = e8m0_code<FMT, RCEIL>(m << 16);
        mu0[i] = e8m0_mult(code);
        sb[p0 + 16 * i] = (uint8_t)code;
      }
    }
    // pass 2: each row unpacked once, cast with both multipliers
    uint8_t* o0 = DIM0 ? q0 + (r0 + rl) * C + c0 + cl : nullptr;
    uint8_t* o1 = DIM1 ? q1 + (r0 + rl) * C + c0 + cl : nullptr;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float2 f[4];
      const uint32_t w[4] = {raw[i].x, raw[i].y, raw[i].z, raw[i].w};
#pragma unroll
      for (int q = 0; q < 4; ++q) f[q] = make_float2(__uint_as_float(w[q] << 16), __uint_as_float(w[q] & 0xFFFF0000u));
      if (DIM0) {
        const float2 mm[4] = {make_float2(mu0[i], mu0[i]), make_float2(mu0[i], mu0[i]), make_float2(mu0[i], mu0[i]),
                              make_float2(mu0[i], mu0[i])};
        *reinterpret_cast<uint2*>(o0 + i * C) = cast8_f32x2<FMT>(f, mm);
      }
      if (DIM1) *reinterpret_cast<uint2*>(o1 + i * C) = cast8_f32x2<FMT>(f, mu1);
    }
    pr0 = r0;
    pc0 = c0;
    if ((int)blockIdx.x + (k + 1) * G >= num_tiles) {   // last tile of this CTA: publish its codes
      asm volatile("bar.sync 1, 256;" ::: "memory");
      store_sf(k & 1, pr0, pc0);
    }
  }
}

// MXFP8 FSDP gather helper: re-tile gathered dim1 E8M0 scales from rank-major order
// [P][Kt][Tl] 512-byte tiles (rank p's shard-local blocked [K, Nl/32] matrix) into the blocked
// layout of the full [K, P*Nl/32] matrix, [Kt][P*Tl] tiles.  One thread per 16-byte unit.
__global__ void __launch_bounds__(256) sf_unshard_kernel(const uint4* __restrict__ in, int P, int64_t Kt, int64_t Tl,
                                                         uint4* __restrict__ out) {
  const int64_t n = (int64_t)P * Kt * Tl * 32;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tile = i >> 5, u = i & 31;
    const int64_t kt = tile / (P * Tl), jc = tile - kt * (P * Tl);
    const int64_t p = jc / Tl, jl = jc - p * Tl;
    out[i] = __ldg(in + ((p * Kt + kt) * Tl + jl) * 32 + u);
  }
}

// ---------------------------------------------------------------------------
// cast_push: the tensorwise cast of an FSDP weight shard fused with the all-gather's data
// movement (PAPER.md:596 enable_fp8_all_gather): each 8-byte group of codes is written straight
// into slot `rank` of every rank's gather buffer over NVLink (peer pointers), so the FP8 bytes
// never round-trip through local HBM and no collective kernel runs.  The last CTA to finish
// (ticket on the local counter) fences at system scope and publishes the epoch to every peer.
// ---------------------------------------------------------------------------
template <typename T, int FMT>
__global__ void __launch_bounds__(256) cast_push_kernel(const T* __restrict__ x, int64_t R, int64_t C, int64_t ld,
                                                        const float* __restrict__ scale,
                                                        const __grid_constant__ P2PPeers pe, int64_t slot_off,
                                                        P2PSig* mine, uint32_t epoch) {
  const int t = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * 128, c0 = (int64_t)blockIdx.x * 128;
  const int vrows = imin128(R - r0), vcols = imin128(C - c0);
  const int cc = (t & 15) * 8;
  const bool cvalid = cc < vcols;
  Raw8<T> raw[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int rr = (t >> 4) + 16 * i;
    if (cvalid && rr < vrows) raw[i].load(x + (r0 + rr) * ld + c0 + cc);
  }
  const float s = __ldg(scale);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int rr = (t >> 4) + 16 * i;
    if (!cvalid || rr >= vrows) continue;
    float v[8];
    raw[i].get(v);
    const uint2 b = cast8<FMT>(v, s);
    const int64_t off = slot_off + (r0 + rr) * C + c0 + cc;
    for (int j = 0; j < pe.P; ++j) {
      int p = pe.rank + j;
      if (p >= pe.P) p -= pe.P;
      *reinterpret_cast<uint2*>(pe.buf[p] + off) = b;
    }
  }
  __syncthreads();
  if (t == 0) {
    __threadfence_system();
    const unsigned total = gridDim.x * gridDim.y;
    if (atomicAdd(&mine->ctas, 1u) == total - 1) {   // every CTA's pushes happen-before this point
      mine->ctas = 0;
      __threadfence_system();
      for (int p = 0; p < pe.P; ++p) st_release_sys_u64(&pe.sig[p]->done[pe.rank], epoch);
    }
  }
}

// FP8 byte transpose [R, C] -> [C, R] (R, C multiples of 16).
__global__ void __launch_bounds__(256) transpose_u8_kernel(const uint8_t* __restrict__ in, int64_t R, int64_t C,
                                                           uint8_t* __restrict__ out) {
  __shared__ __align__(16) uint32_t tile[128 * 32];
  const int t = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * 128, c0 = (int64_t)blockIdx.x * 128;
  const int vrows = imin128(R - r0), vcols = imin128(C - c0);
  const int cc = (t & 15) * 8;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int rr = (t >> 4) + 16 * i;
    if (cc < vcols && rr < vrows)
      *reinterpret_cast<uint2*>(&tile[swz(rr, cc >> 2)]) =
          __ldg(reinterpret_cast<const uint2*>(in + (r0 + rr) * C + c0 + cc));
  }
  __syncthreads();
  store_transposed(tile, out, R, r0, c0, vrows, vcols);
}

// ---------------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------------
static int sm_count() { return device_sm_count(); }
static inline dim3 tile_grid(int64_t R, int64_t C) { return dim3((unsigned)((C + 127) / 128), (unsigned)((R + 127) / 128)); }

// knob amax_tile_tma = 0 selects the register-only amax_tile_kernel (A/B comparisons).
static bool amax_tile_use_tma() { return knob(KNOB_AMAX_TILE_TMA) == 1; }
// knob cast_grid > 0 caps a persistent grid (tests: many tiles per CTA)
static int64_t cap_grid(int64_t cap) {
  const int g = knob(KNOB_CAST_GRID);
  return (g > 0 && g < cap) ? g : cap;
}

template <int MODE>
static cudaError_t amax_tma_go(const CUtensorMap& m, int64_t R, int64_t C, int64_t tiles, uint32_t* at, uint32_t* ar,
                               uint32_t* ac, cudaStream_t st, const Seg& seg, const CUtensorMap* m1 = nullptr,
                               AmaxSecond d = AmaxSecond{}) {
  constexpr int ST = 3;
  constexpr int smem = ST * 128 * 256 + 8 * 128 * 4 + 64 + ST * 8;
  auto kern = amax_tile_tma_kernel<MODE, ST>;
  const cudaError_t attr_err = ensure_smem<amax_tile_tma_kernel<MODE, ST>>(smem);
  if (attr_err != cudaSuccess) return attr_err;
  const int64_t cap = cap_grid((int64_t)sm_count() * 2);
  if (!m1) {
    d = AmaxSecond{};
    d.tiles0 = (int)tiles;
    d.strips0 = (int)(R >> 7);
  }
  const int64_t all = (int64_t)d.tiles0 + d.tiles1;
  LaunchScope ls(K_AMAX, st);
  kern<<<(unsigned)(all < cap ? all : cap), 256, smem, st>>>(m, R, C, at, ar, ac, seg, m1 ? *m1 : m, d);
  return cudaGetLastError();
}

// Row / column amax of n bf16 tensors by one amax_rc launch (outputs pre-zeroed).  cudaErrorNotSupported
// when a shape does not fit the TMA path (rows or columns not multiples of 128, unaligned rows).
cudaError_t launch_amax_rc(const AmaxRCTensor* ts, int n, int mode, cudaStream_t st, const Seg& seg) {
  auto enc = get_encode();
  if (!enc || n < 1 || n > AMAX_RC_MAX || (mode != 2 && mode != 4 && mode != 6)) return cudaErrorNotSupported;
  AmaxRCArgs a{};
  a.n = n;
  a.seg = seg;
  a.dbg = knob(KNOB_AMAX_RC_DEBUG);
  a.sleep = (knob(KNOB_WAIT_SLEEP) & 1) != 0;
  for (int k = 0; k < n; ++k) {
    const AmaxRCTensor& x = ts[k];
    if (x.R <= 0 || x.C <= 0 || x.R % 128 || x.C % 128 || (x.ld * 2) % 16 || (reinterpret_cast<uintptr_t>(x.x) & 15))
      return cudaErrorNotSupported;
    cuuint64_t dims[2] = {(cuuint64_t)x.C, (cuuint64_t)x.R};
    cuuint64_t strides[1] = {(cuuint64_t)x.ld * 2};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t estr[2] = {1, 1};
    if (enc(&a.map[k], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x.x), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorNotSupported;
    const int64_t tr = x.R / 128, tc = x.C / 128;
    if ((int64_t)a.tstart[k] + tr * tc > (int64_t)INT32_MAX) return cudaErrorNotSupported;
    a.tstart[k + 1] = a.tstart[k] + (int)(tr * tc);
    a.tiles_x[k] = (int)tc;
    a.strip0[k] = k ? a.strip0[k - 1] + (int)(ts[k - 1].R / 128) : 0;
    a.C[k] = x.C;
    a.row[k] = x.row;
    a.col[k] = x.col;
    if (((mode & 2) && !x.row) || ((mode & 4) && !x.col)) return cudaErrorInvalidValue;
  }
  constexpr int ST = 3;
  constexpr int smem = ST * 128 * 256 + 1024 + 16 * ST;
  const int64_t all = a.tstart[n];
  const int64_t cap = cap_grid((int64_t)sm_count() * 2);
  const unsigned g = (unsigned)(all < cap ? all : cap);
  cudaError_t e = cudaSuccess;
  LaunchScope ls(K_AMAX, st);
  switch (mode) {
    case 2:
      if ((e = ensure_smem<amax_rc_kernel<2, ST>>(smem)) != cudaSuccess) return e;
      amax_rc_kernel<2, ST><<<g, 288, smem, st>>>(a);
      break;
    case 4:
      if ((e = ensure_smem<amax_rc_kernel<4, ST>>(smem)) != cudaSuccess) return e;
      amax_rc_kernel<4, ST><<<g, 288, smem, st>>>(a);
      break;
    default:
      if ((e = ensure_smem<amax_rc_kernel<6, ST>>(smem)) != cudaSuccess) return e;
      amax_rc_kernel<6, ST><<<g, 288, smem, st>>>(a);
      break;
  }
  return cudaGetLastError();
}

static cudaError_t amax_bulk_go(const void* x0, int64_t b0, uint32_t* out0, const void* x1, int64_t b1, uint32_t* out1,
                                bool bf16, cudaStream_t st);

template <typename T>
static cudaError_t amax_launch_t(const void* x, int64_t R, int64_t C, int64_t ld, int mode, uint32_t* at,
                                 uint32_t* ar, uint32_t* ac, cudaStream_t st, const Seg& seg) {
  const T* p = static_cast<const T*>(x);
  if (mode == 1 && ld == C && knob(KNOB_AMAX_BULK) == 1 && (R * C * (int64_t)sizeof(T)) % 16 == 0)
    return amax_bulk_go(x, R * C * (int64_t)sizeof(T), at, nullptr, 0, nullptr, sizeof(T) == 2, st);
  if (mode == 1 && ld == C) {
    const int64_t n16 = R * C * (int64_t)sizeof(T) / 16;
    // tuning knobs amax_blocks_per_sm / amax_loads (16-byte loads per thread: 4, 8, 12, 16); default
    // 8 / 8 (measured 5.2 TB/s pure read on C2's dY, vs 6.45 TB/s for a read+write copy and 3.0 for torch.amax)
    const int bps = knob(KNOB_AMAX_BLOCKS_PER_SM);
    const int u = knob(KNOB_AMAX_LOADS);
    const int64_t cap = (int64_t)sm_count() * bps;
    const int64_t want = (n16 + 255) / 256;
    const unsigned g = (unsigned)(want < cap ? want : cap);
    const uint4* xv = reinterpret_cast<const uint4*>(x);
    LaunchScope ls(K_AMAX, st);
    const int gi = (int)g;
    if (u == 4) amax_flat_kernel<T, 4><<<g, 256, 0, st>>>(xv, n16, at, xv, 0, at, gi);
    else if (u == 12) amax_flat_kernel<T, 12><<<g, 256, 0, st>>>(xv, n16, at, xv, 0, at, gi);
    else if (u == 16) amax_flat_kernel<T, 16><<<g, 256, 0, st>>>(xv, n16, at, xv, 0, at, gi);
    else amax_flat_kernel<T, 8><<<g, 256, 0, st>>>(xv, n16, at, xv, 0, at, gi);
    return cudaGetLastError();
  }
  const int64_t tiles = ((R + 127) / 128) * ((C + 127) / 128);
  if (sizeof(T) == 2 && mode != 1 && knob(KNOB_AMAX_RC) == 1) {
    const AmaxRCTensor one{x, R, C, ld, ar, ac};
    const cudaError_t e = launch_amax_rc(&one, 1, mode, st, seg);
    if (e != cudaErrorNotSupported) return e;
  }
  if (sizeof(T) == 2 && R % 128 == 0 && C % 128 == 0 && mode != 1 && amax_tile_use_tma()) {
    auto enc = get_encode();
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box[2] = {128, 128};
    cuuint32_t estr[2] = {1, 1};
    if (enc && enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
      switch (mode) {
        case 2: return amax_tma_go<2>(m, R, C, tiles, at, ar, ac, st, seg);
        case 4: return amax_tma_go<4>(m, R, C, tiles, at, ar, ac, st, seg);
        case 6: return amax_tma_go<6>(m, R, C, tiles, at, ar, ac, st, seg);
        default: break;
      }
    }
  }
  const int64_t cap = (int64_t)sm_count() * 8;   // persistent: up to 8 resident CTAs per SM
  dim3 g((unsigned)(tiles < cap ? tiles : cap));
  LaunchScope ls(K_AMAX, st);
  switch (mode) {
    case 1: amax_tile_kernel<T, 1><<<g, 256, 0, st>>>(p, R, C, ld, at, ar, ac, seg); break;
    case 2: amax_tile_kernel<T, 2><<<g, 256, 0, st>>>(p, R, C, ld, at, ar, ac, seg); break;
    case 4: amax_tile_kernel<T, 4><<<g, 256, 0, st>>>(p, R, C, ld, at, ar, ac, seg); break;
    case 6: amax_tile_kernel<T, 6><<<g, 256, 0, st>>>(p, R, C, ld, at, ar, ac, seg); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// Row / column amax of two bf16 tensors (the forward's X and W) in one TMA-ring launch: the second
// tensor's tiles follow the first's in the persistent tile order.  cudaErrorNotSupported when a shape
// does not fit the TMA path (the caller then launches the tensors separately).
cudaError_t launch_amax_dual(const void* x0, int64_t R0, int64_t C0, int64_t ld0, const void* x1, int64_t R1, int64_t C1,
                             int64_t ld1, int mode, uint32_t* ar0, uint32_t* ac0, uint32_t* ar1, uint32_t* ac1,
                             cudaStream_t st) {
  if (knob(KNOB_AMAX_RC) == 1) {
    const AmaxRCTensor two[2] = {{x0, R0, C0, ld0, ar0, ac0}, {x1, R1, C1, ld1, ar1, ac1}};
    return launch_amax_rc(two, 2, mode, st);
  }
  auto enc = get_encode();
  if (!enc || !amax_tile_use_tma() || (mode != 2 && mode != 4 && mode != 6)) return cudaErrorNotSupported;
  const void* xs[2] = {x0, x1};
  const int64_t Rs[2] = {R0, R1}, Cs[2] = {C0, C1}, lds[2] = {ld0, ld1};
  CUtensorMap m[2];
  for (int k = 0; k < 2; ++k) {
    if (Rs[k] % 128 || Cs[k] % 128 || Rs[k] <= 0 || Cs[k] <= 0) return cudaErrorNotSupported;
    cuuint64_t dims[2] = {(cuuint64_t)Cs[k], (cuuint64_t)Rs[k]};
    cuuint64_t strides[1] = {(cuuint64_t)lds[k] * 2};
    cuuint32_t box[2] = {128, 128};
    cuuint32_t estr[2] = {1, 1};
    if (enc(&m[k], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(xs[k]), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorNotSupported;
  }
  AmaxSecond d{};
  d.tiles0 = (int)((R0 / 128) * (C0 / 128));
  d.tiles1 = (int)((R1 / 128) * (C1 / 128));
  d.tiles_x1 = (int)(C1 / 128);
  d.strips0 = (int)(R0 / 128);
  d.amax_row1 = ar1;
  d.amax_col1 = ac1;
  const int64_t tiles = d.tiles0;
  switch (mode) {
    case 2: return amax_tma_go<2>(m[0], R0, C0, tiles, nullptr, ar0, ac0, st, Seg{}, &m[1], d);
    case 4: return amax_tma_go<4>(m[0], R0, C0, tiles, nullptr, ar0, ac0, st, Seg{}, &m[1], d);
    default: return amax_tma_go<6>(m[0], R0, C0, tiles, nullptr, ar0, ac0, st, Seg{}, &m[1], d);
  }
}

cudaError_t launch_amax_multi(const AmaxMultiArgs& a, cudaStream_t st) {
  const int64_t total = a.chunk_start[a.n];
  if (total == 0) return cudaSuccess;
  const int64_t cap = (int64_t)sm_count() * 8 * 8;   // warps: 8 CTAs of 8 warps per SM
  const int64_t warps = total < cap ? total : cap;
  LaunchScope ls(K_AMAX, st);
  amax_multi_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(a);
  return cudaGetLastError();
}

// Tensorwise amax of two contiguous tensors of one dtype in one launch (the forward's X and W): the
// persistent grid is split between them in proportion to their sizes.
// Tensorwise amax of one or two contiguous tensors through 1-D bulk copies (knob amax_bulk): 32 KB chunks
// handed out interleaved over a persistent grid (CTA b: chunks b, b + G, ...; neighbouring chunks are read
// at the same time), ST chunks in flight per CTA landing on mbarriers, |x| max on raw bit patterns, one
// atomic per tensor per CTA.  Chunks [0, c0) belong to x0, [c0, c0 + c1) to x1.
template <typename T, int ST>
__global__ void __launch_bounds__(256) amax_bulk_kernel(const uint8_t* __restrict__ x0, int64_t b0, uint32_t* out0,
                                                        const uint8_t* __restrict__ x1, int64_t b1, uint32_t* out1) {
  constexpr int CH = 32768;
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t s0 = smem_u32(sm), bar0 = s0 + ST * CH;
  const int t = threadIdx.x;
  const int64_t c0 = (b0 + CH - 1) / CH, c1 = (b1 + CH - 1) / CH, total = c0 + c1;
  const int64_t G = gridDim.x;
  auto bytes_of = [&](int64_t id) -> uint32_t {
    const int64_t off = id < c0 ? id * CH : (id - c0) * CH;
    const int64_t n = id < c0 ? b0 : b1;
    return (uint32_t)(n - off < CH ? n - off : CH);
  };
  auto issue = [&](int k) {
    const int64_t id = blockIdx.x + (int64_t)k * G;
    if (id < total) {
      const uint32_t nb = bytes_of(id), bar = bar0 + 8 * (k % ST);
      mbar_arrive_expect_tx(bar, nb);
      bulk_load(s0 + (k % ST) * CH, id < c0 ? x0 + id * CH : x1 + (id - c0) * CH, nb, bar);
    }
  };
  if (t == 0) {
    for (int i = 0; i < ST; ++i) mbar_init(bar0 + 8 * i, 1);
    fence_mbar_init();
    for (int k = 0; k < ST; ++k) issue(k);
  }
  __syncthreads();
  constexpr bool BF = sizeof(T) == 2;
  const uint32_t mask = BF ? 0x7FFF7FFFu : 0x7FFFFFFFu;
  uint32_t m0 = 0, m1 = 0;
  for (int k = 0;; ++k) {
    const int64_t id = blockIdx.x + (int64_t)k * G;
    if (id >= total) break;
    mbar_wait(bar0 + 8 * (k % ST), (uint32_t)(k / ST) & 1u);
    const int nv = (int)(bytes_of(id) / 16);
    const uint4* v = reinterpret_cast<const uint4*>(sm + (k % ST) * CH);
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < CH / 16 / 256; ++i) {
      const int j = t + 256 * i;
      if (j < nv) {
        const uint4 q = v[j];
        if (BF) {
          m = __vmaxu2(m, q.x & mask); m = __vmaxu2(m, q.y & mask);
          m = __vmaxu2(m, q.z & mask); m = __vmaxu2(m, q.w & mask);
        } else {
          m = max(m, q.x & mask); m = max(m, q.y & mask); m = max(m, q.z & mask); m = max(m, q.w & mask);
        }
      }
    }
    if (id < c0) m0 = BF ? __vmaxu2(m0, m) : max(m0, m);
    else m1 = BF ? __vmaxu2(m1, m) : max(m1, m);
    __syncthreads();   // stage consumed by every thread
    if (t == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k + ST);
    }
  }
  if (BF) {   // packed bf16 pairs -> the larger half, as an fp32 bit pattern
    m0 = max(m0 & 0xFFFFu, m0 >> 16) << 16;
    m1 = max(m1 & 0xFFFFu, m1 >> 16) << 16;
  }
  __shared__ uint32_t red[2][8];
  m0 = __reduce_max_sync(0xffffffffu, m0);
  m1 = __reduce_max_sync(0xffffffffu, m1);
  if ((t & 31) == 0) {
    red[0][t >> 5] = m0;
    red[1][t >> 5] = m1;
  }
  __syncthreads();
  if (t == 0) {
    uint32_t a = 0, b = 0;
    for (int w = 0; w < 8; ++w) {
      a = max(a, red[0][w]);
      b = max(b, red[1][w]);
    }
    if (a) atomicMax(out0, a);
    if (b && out1) atomicMax(out1, b);
  }
}

static cudaError_t amax_bulk_go(const void* x0, int64_t b0, uint32_t* out0, const void* x1, int64_t b1, uint32_t* out1,
                                bool bf16, cudaStream_t st) {
  constexpr int ST = 4, CH = 32768;
  constexpr int smem = ST * CH + ST * 8;
  const cudaError_t e = bf16 ? ensure_smem<amax_bulk_kernel<__nv_bfloat16, ST>>(smem)
                             : ensure_smem<amax_bulk_kernel<float, ST>>(smem);
  if (e != cudaSuccess) return e;
  const int64_t chunks = (b0 + CH - 1) / CH + (b1 + CH - 1) / CH;
  const int64_t cap = cap_grid((int64_t)sm_count() * 1);
  const unsigned g = (unsigned)(chunks < cap ? chunks : cap);
  LaunchScope ls(K_AMAX, st);
  const uint8_t* p0 = static_cast<const uint8_t*>(x0);
  const uint8_t* p1 = static_cast<const uint8_t*>(x1);
  if (bf16) amax_bulk_kernel<__nv_bfloat16, ST><<<g, 256, smem, st>>>(p0, b0, out0, p1, b1, out1);
  else amax_bulk_kernel<float, ST><<<g, 256, smem, st>>>(p0, b0, out0, p1, b1, out1);
  return cudaGetLastError();
}

cudaError_t launch_amax_flat_dual(const void* x0, int64_t n0_elems, uint32_t* out0, const void* x1, int64_t n1_elems,
                                  uint32_t* out1, bool bf16, cudaStream_t st) {
  const int es = bf16 ? 2 : 4;
  if ((n0_elems * es) % 16 || (n1_elems * es) % 16 || n0_elems <= 0 || n1_elems <= 0) return cudaErrorNotSupported;
  if (knob(KNOB_AMAX_BULK) == 1) return amax_bulk_go(x0, n0_elems * es, out0, x1, n1_elems * es, out1, bf16, st);
  const int64_t a16 = n0_elems * es / 16, b16 = n1_elems * es / 16;
  const int64_t cap = (int64_t)sm_count() * 8;
  const int64_t want = (a16 + b16 + 255) / 256;
  const int g = (int)(want < cap ? want : cap);
  if (g < 2) return cudaErrorNotSupported;
  int g0 = (int)((double)g * (double)a16 / (double)(a16 + b16) + 0.5);
  g0 = g0 < 1 ? 1 : (g0 > g - 1 ? g - 1 : g0);
  const uint4* v0 = reinterpret_cast<const uint4*>(x0);
  const uint4* v1 = reinterpret_cast<const uint4*>(x1);
  LaunchScope ls(K_AMAX, st);
  if (bf16) amax_flat_kernel<__nv_bfloat16, 8><<<g, 256, 0, st>>>(v0, a16, out0, v1, b16, out1, g0);
  else amax_flat_kernel<float, 8><<<g, 256, 0, st>>>(v0, a16, out0, v1, b16, out1, g0);
  return cudaGetLastError();
}

cudaError_t launch_amax(const void* x, bool bf16, int64_t R, int64_t C, int64_t ld, int mode, uint32_t* at,
                        uint32_t* ar, uint32_t* ac, cudaStream_t st, const Seg& seg) {
  return bf16 ? amax_launch_t<__nv_bfloat16>(x, R, C, ld, mode, at, ar, ac, st, seg)
              : amax_launch_t<float>(x, R, C, ld, mode, at, ar, ac, st, seg);
}

template <typename T, int FMT>
static cudaError_t cast_launch_t(const void* x, int64_t R, int64_t C, int64_t ld, int qm, int tm,
                                 const float* aq, const float* at, uint8_t* q, uint8_t* qt, float* sq, float* st,
                                 cudaStream_t s, const Seg& seg) {
  const T* p = static_cast<const T*>(x);
  dim3 g = tile_grid(R, C);
#define FP8T_CAST(QM, TM)                                                                       \
  if (qm == QM && tm == TM) {                                                                   \
    LaunchScope ls(K_CAST, s);                                                                  \
    cast_tile_kernel<T, FMT, QM, TM><<<g, 256, 0, s>>>(p, R, C, ld, aq, at, q, qt, sq, st, seg);\
    return cudaGetLastError();                                                                  \
  }
  FP8T_CAST(1, 0) FP8T_CAST(0, 1) FP8T_CAST(1, 1)
  FP8T_CAST(2, 0) FP8T_CAST(0, 2) FP8T_CAST(2, 2)
  FP8T_CAST(3, 0) FP8T_CAST(0, 3) FP8T_CAST(3, 3)
  FP8T_CAST(2, 3) FP8T_CAST(2, 5) FP8T_CAST(0, 5)
#undef FP8T_CAST
  return cudaErrorInvalidValue;
}

// Rowwise (qm 2, tm 5) casts of bf16 tensors by cast_rc_tma_kernel; cudaErrorNotSupported when a tensor does
// not fit the TMA path (the caller then launches the tile kernel).
// Policy (knob cast_rc_tma): 1 = auto, launches of at most 12288 tiles (c3: every cast but the w1/w3 dY and the w2
// X, W ones -- with two loads in flight per CTA the persistent kernel streams large tensors slower than the
// 8-CTAs-per-SM tile kernel, but it saves the small launches' ramp and tail); 2 = always; 0 = never.
static cudaError_t cast_rc_tma_launch(const CastMulti& m, int fmt, cudaStream_t s) {
  auto enc = get_encode();
  const int pol = knob(KNOB_CAST_RC_TMA);
  if (!enc || pol == 0) return cudaErrorNotSupported;
  if (pol == 1) {
    int64_t tiles = 0;
    for (int k = 0; k < m.n; ++k) tiles += ((m.R[k] + 127) / 128) * ((m.C[k] + 127) / 128);
    if (tiles > 12288) return cudaErrorNotSupported;
  }
  CastRCArgs a{};
  a.n = m.n;
  for (int k = 0; k < m.n; ++k) {
    const int64_t R = m.R[k], C = m.C[k], ld = m.ld[k];
    if (R <= 0 || C <= 0 || R % 128 || C % 128 || (ld * 2) % 16 || !m.q[k] || !m.qt[k] ||
        (reinterpret_cast<uintptr_t>(m.x[k]) & 15) || (reinterpret_cast<uintptr_t>(m.q[k]) & 15) ||
        (reinterpret_cast<uintptr_t>(m.qt[k]) & 15))
      return cudaErrorNotSupported;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
    cuuint64_t sin[1] = {(cuuint64_t)ld * 2}, sout[1] = {(cuuint64_t)C};
    cuuint32_t box[2] = {128, 128};
    cuuint32_t estr[2] = {1, 1};
    if (enc(&a.in[k], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(m.x[k]), dims, sin, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
        enc(&a.oq[k], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, m.q[k], dims, sout, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
        enc(&a.ot[k], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, m.qt[k], dims, sout, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorNotSupported;
    const int64_t tiles = (R / 128) * (C / 128);
    if ((int64_t)a.tstart[k] + tiles > (int64_t)INT32_MAX) return cudaErrorNotSupported;
    a.tstart[k + 1] = a.tstart[k] + (int)tiles;
    a.tiles_x[k] = (int)(C / 128);
    a.amax_q[k] = m.amax_q[k];
    a.amax_t[k] = m.amax_t[k];
    a.scale_q[k] = m.scale_q[k];
    a.scale_t[k] = m.scale_t[k];
  }
  const int64_t all = a.tstart[a.n];
  if (all == 0) return cudaSuccess;
  cudaError_t e;
  LaunchScope ls(K_CAST, s);
  if (knob(KNOB_CAST_RC_WIDE) == 1) {   // 1 CTA of 512 threads per SM, 5-deep ring (four loads in flight)
    constexpr int ST = 5;
    constexpr int smem = ST * 128 * 256 + 1024 + 8 * ST;
    const int64_t cap = cap_grid((int64_t)sm_count());
    const unsigned g = (unsigned)(all < cap ? all : cap);
    if (fmt == 0) {
      if ((e = ensure_smem<cast_rc_tma_kernel<0, ST, 512>>(smem)) != cudaSuccess) return e;
      cast_rc_tma_kernel<0, ST, 512><<<g, 512, smem, s>>>(a);
    } else {
      if ((e = ensure_smem<cast_rc_tma_kernel<1, ST, 512>>(smem)) != cudaSuccess) return e;
      cast_rc_tma_kernel<1, ST, 512><<<g, 512, smem, s>>>(a);
    }
    return cudaGetLastError();
  }
  constexpr int ST = 3;
  constexpr int smem = ST * 128 * 256 + 1024 + 8 * ST;
  const int64_t cap = cap_grid((int64_t)sm_count() * 2);
  const unsigned g = (unsigned)(all < cap ? all : cap);
  if (fmt == 0) {
    if ((e = ensure_smem<cast_rc_tma_kernel<0, ST, 256>>(smem)) != cudaSuccess) return e;
    cast_rc_tma_kernel<0, ST, 256><<<g, 256, smem, s>>>(a);
  } else {
    if ((e = ensure_smem<cast_rc_tma_kernel<1, ST, 256>>(smem)) != cudaSuccess) return e;
    cast_rc_tma_kernel<1, ST, 256><<<g, 256, smem, s>>>(a);
  }
  return cudaGetLastError();
}

template <typename T, int FMT>
static cudaError_t cast_dual_launch_t(const CastMulti& a, int qm, int tm, cudaStream_t s) {
  const unsigned g = (unsigned)a.tstart[a.n];
  if (g == 0) return cudaSuccess;
#define FP8T_CAST2(QM, TM)                                                          \
  if (qm == QM && tm == TM) {                                                       \
    LaunchScope ls(K_CAST, s);                                                      \
    cast_tile_dual_kernel<T, FMT, QM, TM><<<g, 256, 0, s>>>(a);                      \
    return cudaGetLastError();                                                      \
  }
  FP8T_CAST2(1, 0) FP8T_CAST2(2, 5) FP8T_CAST2(2, 0)
#undef FP8T_CAST2
  return cudaErrorInvalidValue;
}

cudaError_t launch_cast_dual(CastMulti a, bool bf16, int fmt, int qm, int tm, cudaStream_t s) {
  if (a.n == 0) a.n = 2;
  if (a.n < 1 || a.n > CAST_MULTI_MAX) return cudaErrorInvalidValue;
  a.tstart[0] = 0;
  for (int k = 0; k < a.n; ++k) {
    const int64_t tiles = ((a.R[k] + 127) / 128) * ((a.C[k] + 127) / 128);
    if (a.tstart[k] + tiles > (int64_t)INT32_MAX) return cudaErrorInvalidValue;
    a.tstart[k + 1] = a.tstart[k] + (int)tiles;
  }
  if (bf16 && qm == 2 && tm == 5) {
    const cudaError_t e = cast_rc_tma_launch(a, fmt, s);
    if (e != cudaErrorNotSupported) return e;
  }
  if (bf16)
    return fmt == 0 ? cast_dual_launch_t<__nv_bfloat16, 0>(a, qm, tm, s) : cast_dual_launch_t<__nv_bfloat16, 1>(a, qm, tm, s);
  return fmt == 0 ? cast_dual_launch_t<float, 0>(a, qm, tm, s) : cast_dual_launch_t<float, 1>(a, qm, tm, s);
}

cudaError_t launch_cast(const void* x, bool bf16, int fmt, int64_t R, int64_t C, int64_t ld, int qm, int tm,
                        const float* aq, const float* at, uint8_t* q, uint8_t* qt, float* sq, float* st,
                        cudaStream_t s, const Seg& seg) {
  if (bf16 && qm == 2 && tm == 5 && !seg.offs && seg.seg_rows <= 0) {
    CastMulti m{};
    m.n = 1;
    m.x[0] = x; m.R[0] = R; m.C[0] = C; m.ld[0] = ld; m.amax_q[0] = aq; m.amax_t[0] = at;
    m.q[0] = q; m.qt[0] = qt; m.scale_q[0] = sq; m.scale_t[0] = st;
    const cudaError_t e = cast_rc_tma_launch(m, fmt, s);
    if (e != cudaErrorNotSupported) return e;
  }
  if (bf16)
    return fmt == 0 ? cast_launch_t<__nv_bfloat16, 0>(x, R, C, ld, qm, tm, aq, at, q, qt, sq, st, s, seg)
                    : cast_launch_t<__nv_bfloat16, 1>(x, R, C, ld, qm, tm, aq, at, q, qt, sq, st, s, seg);
  return fmt == 0 ? cast_launch_t<float, 0>(x, R, C, ld, qm, tm, aq, at, q, qt, sq, st, s, seg)
                  : cast_launch_t<float, 1>(x, R, C, ld, qm, tm, aq, at, q, qt, sq, st, s, seg);
}

template <typename T, int FMT, bool RC>
static cudaError_t mx_launch_t(const void* x, int64_t R, int64_t C, int64_t ld, uint8_t* q0, uint8_t* sf0,
                               uint8_t* q1, uint8_t* sf1, bool tr1, cudaStream_t s) {
  const T* p = static_cast<const T*>(x);
  dim3 g = tile_grid(R, C);
  LaunchScope ls(K_MX, s);
  if (q0 && q1) {
    if (tr1) mx_cast_kernel<T, FMT, RC, true, true, true><<<g, 256, 0, s>>>(p, R, C, ld, q0, sf0, q1, sf1);
    else mx_cast_kernel<T, FMT, RC, true, true, false><<<g, 256, 0, s>>>(p, R, C, ld, q0, sf0, q1, sf1);
  } else if (q0) {
    mx_cast_kernel<T, FMT, RC, true, false, true><<<g, 256, 0, s>>>(p, R, C, ld, q0, sf0, q1, sf1);
  } else {
    if (tr1) mx_cast_kernel<T, FMT, RC, false, true, true><<<g, 256, 0, s>>>(p, R, C, ld, q0, sf0, q1, sf1);
    else mx_cast_kernel<T, FMT, RC, false, true, false><<<g, 256, 0, s>>>(p, R, C, ld, q0, sf0, q1, sf1);
  }
  return cudaGetLastError();
}

template <int FMT, bool RC, bool D0, bool D1, bool TR, int ST, bool TS = false>
static cudaError_t mx_tma_go(const CUtensorMap& m, int64_t R, int64_t C, uint8_t* q0, uint8_t* sf0, uint8_t* q1,
                             uint8_t* sf1, cudaStream_t s) {
  auto kern = mx_cast_tma_kernel<FMT, RC, D0, D1, TR, ST, TS>;
  constexpr int smem = MxSmem<ST, TR>::BYTES;
  const cudaError_t attr_err = ensure_smem<mx_cast_tma_kernel<FMT, RC, D0, D1, TR, ST, TS>>(smem);
  if (attr_err != cudaSuccess) return attr_err;
  CUtensorMap mq0 = m, mq1 = m;
  if (TS) {   // u8 [R, C] code maps, 128 x 128 boxes
    auto enc = get_encode();
    if (!enc) return cudaErrorNotSupported;
    uint8_t* qs[2] = {q0, q1};
    CUtensorMap* ms[2] = {&mq0, &mq1};
    for (int j = 0; j < 2; ++j) {
      cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
      cuuint64_t strides[1] = {(cuuint64_t)C};
      cuuint32_t box[2] = {128, 128};
      cuuint32_t estr[2] = {1, 1};
      if (enc(ms[j], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, qs[j], dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    }
  }
  const int64_t tiles = (R >> 7) * (C >> 7);
  const int64_t cap = cap_grid((int64_t)sm_count() * (TR ? 1 : (ST == 2 ? 3 : 2)));
  LaunchScope ls(K_MX, s);
  kern<<<(unsigned)(tiles < cap ? tiles : cap), 256, smem, s>>>(m, R, C, q0, sf0, q1, sf1, knob(KNOB_MX_CAST_DEBUG), mq0, mq1);
  return cudaGetLastError();
}

template <int FMT, bool RC, bool D0, bool D1>
static cudaError_t mx_ws_go(const CUtensorMap& m, int64_t R, int64_t C, uint8_t* q0, uint8_t* sf0, uint8_t* q1,
                            uint8_t* sf1, cudaStream_t s) {
  constexpr int ST = 3;
  constexpr int smem = ST * 128 * 256 + 2048 + 16 * ST;
  const cudaError_t attr_err = ensure_smem<mx_cast_ws_kernel<FMT, RC, D0, D1, ST>>(smem);
  if (attr_err != cudaSuccess) return attr_err;
  const int64_t tiles = (R >> 7) * (C >> 7);
  const int64_t cap = cap_grid((int64_t)sm_count() * 2);
  LaunchScope ls(K_MX, s);
  mx_cast_ws_kernel<FMT, RC, D0, D1, ST><<<(unsigned)(tiles < cap ? tiles : cap), 288, smem, s>>>(m, R, C, q0, sf0, q1, sf1,
                                                                                          knob(KNOB_WAIT_SLEEP) & 1);
  return cudaGetLastError();
}

template <int FMT, bool RC>
static cudaError_t mx_tma_launch_t(const void* x, int64_t R, int64_t C, int64_t ld, uint8_t* q0, uint8_t* sf0,
                                   uint8_t* q1, uint8_t* sf1, bool tr1, cudaStream_t s) {
  auto enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {128, 128};
  cuuint32_t estr[2] = {1, 1};
  if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  if (!tr1 && knob(KNOB_MX_CAST_WS) == 1 && knob(KNOB_MX_CAST_OCC3) == 0 && knob(KNOB_MX_CAST_DEBUG) == 0) {
    if (q0 && q1) return mx_ws_go<FMT, RC, true, true>(m, R, C, q0, sf0, q1, sf1, s);
    if (q0) return mx_ws_go<FMT, RC, true, false>(m, R, C, q0, sf0, q1, sf1, s);
    return mx_ws_go<FMT, RC, false, true>(m, R, C, q0, sf0, q1, sf1, s);
  }
  if (q0 && q1) {
    if (tr1) return mx_tma_go<FMT, RC, true, true, true, 4>(m, R, C, q0, sf0, q1, sf1, s);
    if (knob(KNOB_MX_CAST_OCC3) == 1) return mx_tma_go<FMT, RC, true, true, false, 2>(m, R, C, q0, sf0, q1, sf1, s);
    if (knob(KNOB_MX_CAST_TSTORE) == 1 && knob(KNOB_MX_CAST_DEBUG) == 0 && (reinterpret_cast<uintptr_t>(q0) & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(q1) & 15) == 0 && C % 16 == 0)
      return mx_tma_go<FMT, RC, true, true, false, 3, true>(m, R, C, q0, sf0, q1, sf1, s);
    return mx_tma_go<FMT, RC, true, true, false, 3>(m, R, C, q0, sf0, q1, sf1, s);
  }
  if (q0) return mx_tma_go<FMT, RC, true, false, false, 3>(m, R, C, q0, sf0, q1, sf1, s);
  if (tr1) return mx_tma_go<FMT, RC, false, true, true, 4>(m, R, C, q0, sf0, q1, sf1, s);
  return mx_tma_go<FMT, RC, false, true, false, 3>(m, R, C, q0, sf0, q1, sf1, s);
}

// knob mx_cast_tma = 0 selects the register-only mx_cast_kernel (A/B comparisons; fp32 inputs always use it).
static bool mx_use_tma() { return knob(KNOB_MX_CAST_TMA) == 1; }

cudaError_t launch_mx_cast(const void* x, bool bf16, int fmt, bool rceil, int64_t R, int64_t C, int64_t ld,
                           uint8_t* q0, uint8_t* sf0, uint8_t* q1, uint8_t* sf1, cudaStream_t s, bool tr1) {
  if (bf16 && mx_use_tma()) {
    if (fmt == 0) return rceil ? mx_tma_launch_t<0, true>(x, R, C, ld, q0, sf0, q1, sf1, tr1, s)
                               : mx_tma_launch_t<0, false>(x, R, C, ld, q0, sf0, q1, sf1, tr1, s);
    return rceil ? mx_tma_launch_t<1, true>(x, R, C, ld, q0, sf0, q1, sf1, tr1, s)
                 : mx_tma_launch_t<1, false>(x, R, C, ld, q0, sf0, q1, sf1, tr1, s);
  }
#define FP8T_MX(T)                                                                                  \
  if (fmt == 0) return rceil ? mx_launch_t<T, 0, true>(x, R, C, ld, q0, sf0, q1, sf1, tr1, s)       \
                             : mx_launch_t<T, 0, false>(x, R, C, ld, q0, sf0, q1, sf1, tr1, s);     \
  return rceil ? mx_launch_t<T, 1, true>(x, R, C, ld, q0, sf0, q1, sf1, tr1, s)                     \
               : mx_launch_t<T, 1, false>(x, R, C, ld, q0, sf0, q1, sf1, tr1, s);
  if (bf16) { FP8T_MX(__nv_bfloat16) }
  FP8T_MX(float)
#undef FP8T_MX
}

cudaError_t launch_sf_unshard(const uint8_t* in, int P, int64_t Kt, int64_t Tl, uint8_t* out, cudaStream_t s) {
  const int64_t n = (int64_t)P * Kt * Tl * 32;
  if (n == 0) return cudaSuccess;
  const int64_t cap = (int64_t)sm_count() * 8, want = (n + 255) / 256;
  LaunchScope ls(K_TRANSPOSE, s);
  sf_unshard_kernel<<<(unsigned)(want < cap ? want : cap), 256, 0, s>>>(reinterpret_cast<const uint4*>(in), P, Kt, Tl,
                                                                        reinterpret_cast<uint4*>(out));
  return cudaGetLastError();
}

cudaError_t launch_cast_push(const void* x, bool bf16, int fmt, int64_t R, int64_t C, int64_t ld, const float* scale,
                             const P2PPeers& pe, int64_t slot_off, P2PSig* mine, uint32_t epoch, cudaStream_t s) {
  const dim3 g = tile_grid(R, C);
  LaunchScope ls(K_CAST, s);
  if (bf16) {
    if (fmt == 0) cast_push_kernel<__nv_bfloat16, 0><<<g, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x), R, C, ld, scale, pe, slot_off, mine, epoch);
    else cast_push_kernel<__nv_bfloat16, 1><<<g, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x), R, C, ld, scale, pe, slot_off, mine, epoch);
  } else {
    if (fmt == 0) cast_push_kernel<float, 0><<<g, 256, 0, s>>>(static_cast<const float*>(x), R, C, ld, scale, pe, slot_off, mine, epoch);
    else cast_push_kernel<float, 1><<<g, 256, 0, s>>>(static_cast<const float*>(x), R, C, ld, scale, pe, slot_off, mine, epoch);
  }
  return cudaGetLastError();
}

cudaError_t launch_transpose_u8(const uint8_t* in, int64_t R, int64_t C, uint8_t* out, cudaStream_t s) {
  LaunchScope ls(K_TRANSPOSE, s);
  transpose_u8_kernel<<<tile_grid(R, C), 256, 0, s>>>(in, R, C, out);
  return cudaGetLastError();
}

}  // namespace fp8t
