/*
 * fp8train.h -- C-ABI of the B200-native dynamically scaled Float8Linear step.
 *
 * Source of the operations: TorchAO (arXiv 2507.16099) §2.1 "FP8 Training"
 * and Appendix A "TorchAO FP8 Scaling Recipes"
 * (PAPER.md:592-599); MX formats from Appendix E.  The paper
 * defines the recipes in prose; the exact arithmetic each call performs is
 * written out in DESIGN.md "Readings" (mirrors SURVEY.md §8c) and
 * cross-referenced below as R-cN.
 *
 * Conventions shared by every call
 * --------------------------------
 *  - All tensor pointers are DEVICE pointers (except where a parameter is
 *    documented as host).  Every compute call is asynchronous on `stream`
 *    (a cudaStream_t passed as void*; NULL = legacy default stream) and never
 *    synchronises the host.  amax and scales live in device memory only
 *    (dynamic scaling).
 *  - Ownership: the caller owns every buffer.  The library never allocates or
 *    frees device memory inside these calls; temporaries come from the
 *    caller's workspace, sized by the *_bytes() helpers.
 *  - Errors: argument, shape and alignment checks run BEFORE any launch and
 *    return a status with no partial work.  Launch failures -> FP8_ECUDA,
 *    NCCL failures -> FP8_ENCCL.  Asynchronous device faults surface at the
 *    caller's next synchronisation, as usual in CUDA.  fp8_last_error()
 *    returns a thread-local message for the last non-OK status.
 *  - Layout: every matrix is row-major with a leading dimension `ld` in
 *    elements.  FP8 code buffers (`q`, `q_t`) are dense (ld = cols, resp.
 *    ld = rows for the transposed copy).
 *  - Alignment: pointers 16-byte aligned; rows, cols >= 16 and multiples of
 *    16; ld * element_size a multiple of 16.  MX (block-32) operands need
 *    rows and cols multiples of 128 (the E8M0 blocked layout below).
 *    Violations -> FP8_EALIGN.
 *  - Inputs must be finite (PAPER.md:281 recipes assume it; R-c9).  NaN
 *    propagates through amax; it is not detected.
 *  - Thread safety: re-entrant; no mutable global state beyond per-device
 *    cached attributes (SM count, shared-memory limits), the lazily resolved
 *    cuTensorMapEncodeTiled entry point, the thread-local error string, the
 *    kernel-variant knobs (fp8_set_knob), and the GEMM tile scheduler's
 *    counters: a module-global device array of 2 x 4096 slots per device (no
 *    allocation in any call).  Each eager GEMM launch takes the next slot of
 *    the first region (atomic round robin) and resets it when its last CTA
 *    pair has fetched its last tile; more than 4096 GEMM launches executing
 *    concurrently would share slots (stream-ordered launches never do).  A GEMM
 *    captured into a CUDA graph takes a slot of the second region for good
 *    (kept on every replay, never handed out again); after 4096 captured GEMMs
 *    on a device, further captures use the static tile schedule.  Replays of
 *    one captured graph (or of two execs instantiated from it) must therefore
 *    not execute concurrently.
 *
 * Number formats (R-c1, R-c2, R-c10, R-c11)
 *  - FP8_E4M3: "FN" variant, no inf, NaN 0x7F/0xFF, max 448.
 *  - FP8_E5M2: IEEE-like, inf 0x7C/0xFC, max 57344.
 *  - cast = satRNE(RN32(x * s)): the fp32 product rounded first, then round to
 *    nearest even with saturation to +-max; sign preserved (-0 -> 0x80);
 *    subnormals kept.
 *  - scale s = RN32(fmax / max(amax, 1e-12f)) (multiplicative, fp8 ~= x*s;
 *    R-c3, R-c5, R-c6).  GEMM epilogues multiply by 1/s.
 *  - E8M0 (MX): code c -> 2^(c-127).  FLOOR: c = clamp(floor(log2 amax) -
 *    emax + 127, 0, 254) (emax 8 for e4m3, 15 for e5m2); RCEIL: c =
 *    clamp(127 + ceil(log2(amax / fmax)), 0, 254); zero block -> 0
 *    (R-c12, R-c13).  Elements: satRNE(RN32(x * 2^(127-c))).
 *
 * E8M0 blocked scale layout (MX operands)
 *  The codes of an MX operand with R rows and C columns (blocks of 32 along
 *  the columns) form a logical [R, C/32] byte matrix.  It is stored tiled in
 *  128 x 4 tiles, tiles row-major: tile (rb, cb) starts at byte
 *  (rb * (C/128) + cb) * 512, and inside a tile logical (r, c) sits at byte
 *  (r % 32) * 16 + (r / 32) * 4 + c, r in [0,128), c in [0,4).  This is the
 *  scale-factor atom tcgen05.mma.kind::mxf8f6f4.block_scale consumes from
 *  TMEM (32 lanes x 4 words, replicated per lane quadrant), so the GEMM can
 *  stream it with one bulk copy per tile.  Size: R * C / 32 bytes.
 */
#ifndef FP8TRAIN_H_
#define FP8TRAIN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FP8TRAIN_ABI_VERSION 7

typedef enum {
  FP8_OK = 0,
  FP8_EINVAL = 1,        /* bad argument or shape */
  FP8_EALIGN = 2,        /* alignment / divisibility rule violated */
  FP8_EUNSUPPORTED = 3,  /* valid request this build does not implement */
  FP8_ECUDA = 4,         /* a CUDA runtime/driver call or launch failed */
  FP8_ENCCL = 5,         /* an NCCL call failed */
  FP8_EWORKSPACE = 6     /* workspace smaller than *_workspace_bytes() */
} fp8_status_t;

typedef enum { FP8_DT_F32 = 0, FP8_DT_BF16 = 1 } fp8_dtype_t;
typedef enum { FP8_E4M3 = 0, FP8_E5M2 = 1 } fp8_format_t;

/* Scaling granularity (Appendix A; MX: PAPER.md:735). */
typedef enum {
  FP8_GRAN_TENSOR = 0,   /* one scale for the tensor (tensorwise recipe) */
  FP8_GRAN_ROW = 1,      /* one scale per row, reduced over the columns */
  FP8_GRAN_COL = 2,      /* one scale per column, reduced over the rows */
  FP8_GRAN_ROW_COL = 3,  /* rowwise recipe dual cast from one input: q with per-row
                            scales, q_t with per-column scales */
  FP8_GRAN_MX32 = 4,     /* MXFP8: q = blocks of 32 along columns ("dim0"),
                            q_t = blocks of 32 along rows ("dim1"), E8M0 scales */
  FP8_GRAN_MX32_RM = 5   /* as MX32, but q_t (dim1) is written in the input's layout
                            [rows, cols] instead of transposed: same codes, no transpose;
                            fp8_gemm reads it as an MN-major operand */
} fp8_gran_t;

typedef enum { FP8_MX_FLOOR = 0, FP8_MX_RCEIL = 1 } fp8_mx_round_t;

typedef enum {
  FP8_RECIPE_TENSORWISE = 0,
  FP8_RECIPE_ROWWISE = 1,
  FP8_RECIPE_MXFP8 = 2,          /* PAPER.md:735 (MX formats for training) */
  FP8_RECIPE_ROWWISE_GW_HP = 3   /* rowwise, but dL/dW stays in bfloat16 */
} fp8_recipe_t;

/* High-precision input matrix: row-major, `ld` in elements (cols <= ld <= 2^25; rows, cols multiples of 16
 * in [16, 2^31]; 16-byte aligned pointer and ld * elem_size; FP8_EINVAL / FP8_EALIGN otherwise). */
typedef struct {
  const void* ptr;
  fp8_dtype_t dtype;
  int64_t rows, cols, ld;
} fp8_hp_t;

/* A quantised tensor produced by fp8_cast_scaled (caller-owned buffers).
 *   q      : codes [rows, cols] row-major, or NULL
 *   q_t    : codes of the transposed copy [cols, rows] row-major, or NULL
 *            (MX32_RM: the dim1 codes [rows, cols] row-major, not transposed)
 *   scale  : scales that go with q:
 *              TENSOR float[1], ROW float[rows], COL float[cols],
 *              ROW_COL float[rows] (row scales), MX32 E8M0 blocked [rows x cols/32]
 *   scale_t: scales that go with q_t:
 *              TENSOR/ROW/COL: may alias `scale` or be NULL (same values),
 *              ROW_COL float[cols] (column scales),
 *              MX32 / MX32_RM E8M0 blocked [cols x rows/32]
 *   amax   : float[ ] amax behind `scale` (same shape), or NULL
 *   amax_t : float[ ] amax behind `scale_t` (ROW_COL: [cols]), or NULL
 * For MX32 amax/amax_t are unused (the block amax is fused into the cast). */
typedef struct {
  uint8_t* q;
  uint8_t* q_t;
  void* scale;
  void* scale_t;
  float* amax;
  float* amax_t;
  fp8_format_t fmt;
  fp8_gran_t gran;
  int64_t rows, cols;
} fp8_tensor_t;

/* Linear configuration (Appendix A recipes). */
typedef struct {
  fp8_recipe_t recipe;
  fp8_format_t fmt_fwd;   /* X and W codes: FP8_E4M3 by default (R-c8) */
  fp8_format_t fmt_grad;  /* dY codes: FP8_E5M2 by default (R-c8, R-c14) */
  fp8_mx_round_t mx_round;/* MXFP8 shared-exponent rule (R-c12) */
  fp8_dtype_t out_dtype;  /* FP8_DT_BF16 (north star) or FP8_DT_F32 */
} fp8_linear_cfg_t;

/* ---------------------------------------------------------------------------
 * fp8_amax -- amax = max |x| over the scaling unit (R-c step 3).
 *   gran TENSOR -> amax_out float[1]; ROW -> float[rows]; COL -> float[cols].
 *   (ROW_COL / MX32 -> FP8_EINVAL: their amax is fused into the cast.)
 *   Exact: computed as an unsigned max over |x| bit patterns.
 *   `ws` must hold fp8_amax_workspace_bytes() bytes (u32 accumulators).
 * ------------------------------------------------------------------------- */
size_t fp8_amax_workspace_bytes(fp8_hp_t x, fp8_gran_t gran);
fp8_status_t fp8_amax(fp8_hp_t x, fp8_gran_t gran, float* amax_out,
                      void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * fp8_amax_multi -- tensorwise amax of n tensors in ONE launch (SURVEY §8f.2:
 * the weights' amax after the optimizer step, computed together instead of one
 * pass per weight).  xs: HOST array of n descriptors (read during the call);
 * amax_out: device float[n], amax_out[t] = max |xs[t]| (exact, as fp8_amax).
 * 1 <= n <= 48 (FP8_AMAX_MULTI_MAX) per call; no workspace.
 * ------------------------------------------------------------------------- */
#define FP8_AMAX_MULTI_MAX 48
fp8_status_t fp8_amax_multi(const fp8_hp_t* xs, int n, float* amax_out, void* stream);

/* ---------------------------------------------------------------------------
 * fp8_cast_scaled -- scale from amax, then saturating RNE cast (PAPER.md:281-287,
 * Appendix A).  Writes out->q and/or out->q_t (at least one non-NULL), the
 * scales and (optionally) the amax, per out->gran (see fp8_tensor_t).
 *   amax_in: optional precomputed amax (device, TENSOR float[1] only -- e.g. the
 *            all-reduced global weight amax of fp8_fsdp_allgather); NULL = compute.
 *   mx_round: used for FP8_GRAN_MX32 only.
 *   `ws` must hold fp8_cast_workspace_bytes() bytes.
 * out->rows/cols must equal x.rows/cols.
 * ------------------------------------------------------------------------- */
size_t fp8_cast_workspace_bytes(fp8_hp_t x, fp8_gran_t gran);
fp8_status_t fp8_cast_scaled(fp8_hp_t x, fp8_mx_round_t mx_round, const float* amax_in,
                             fp8_tensor_t* out, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * fp8_gemm -- the scaled FP8 GEMM on tcgen05 tensor cores:
 *   D[m,n] = sum_k dec(A[m,k]) dec(B[n,k]) * (1/sa) * (1/sb)   fp32 accumulate
 * Operand storage (`major_a`, `major_b`):
 *   FP8_K_MAJOR : A stored [M,K] row-major (lda >= K); B stored [N,K] (ldb >= K)
 *   FP8_MN_MAJOR: A stored [K,M] row-major (lda >= M); B stored [K,N] (ldb >= N)
 *   (MN-major lets the backward GEMMs read the forward's row-major codes directly,
 *    with no transposed copy; ld in bytes == elements.)
 * Scale modes:
 *   gran TENSOR: sa, sb float[1] (multiplicative scales, device)
 *   gran ROW   : sa float[M], sb float[N]
 *   gran MX32  : sa, sb E8M0 blocked codes of A [M x K/32] and B [N x K/32];
 *                the per-32-block 2^(c-127) factors are applied inside the MMA
 *                (either operand major; the codes' logical layout is unchanged).
 * D is [M,N] row-major with leading dimension ldd elements, dtype out_dtype
 * (BF16 = RN of the fp32 result; F32 = the fp32 result).  Order of the fp32
 * accumulation and of the epilogue products is unspecified (R-c16).
 * ------------------------------------------------------------------------- */
typedef enum { FP8_K_MAJOR = 0, FP8_MN_MAJOR = 1 } fp8_major_t;
fp8_status_t fp8_gemm(const uint8_t* A, fp8_format_t fmt_a, fp8_major_t major_a, const void* sa,
                      const uint8_t* B, fp8_format_t fmt_b, fp8_major_t major_b, const void* sb,
                      fp8_gran_t gran, int64_t M, int64_t N, int64_t K,
                      int64_t lda, int64_t ldb, void* D, fp8_dtype_t out_dtype, int64_t ldd,
                      void* stream);

/* ---------------------------------------------------------------------------
 * Float8Linear forward: Y = X W^T with the recipe's casts (Appendix A):
 *   tensorwise: X, W one scale each;  rowwise: X per row, W per row (over K);
 *   mxfp8: X, W blocks of 32 along K.
 * x [M,K], w [N,K] high precision; y [M,N] out_dtype, dense (ld = N).
 * w_fp8 (nullable): pre-cast weight; then `w` may have ptr NULL (its rows/cols still give
 *   the shape).  tensorwise (e.g. from fp8_fsdp_allgather): w_fp8->q [N,K] codes +
 *   w_fp8->scale float[1].  mxfp8 (e.g. from fp8_fsdp_allgather_mx): gran FP8_GRAN_MX32_RM,
 *   q + scale (dim0) for the forward, q_t + scale_t (dim1) for the backward's dX (the
 *   forward then saves nothing for W).  Other recipes: FP8_EUNSUPPORTED.
 * saved: caller buffer of fp8_linear_saved_bytes() bytes; the forward writes
 *   the FP8 operands the backward needs (the X operand of dW and the W operand
 *   of dX with their scales, per the operand plan of DESIGN.md §2).  Tensorwise
 *   saves the row-major codes the forward GEMM used (the backward GEMMs read
 *   them MN-major); rowwise saves column-scaled copies, MXFP8 dim1 copies.
 * ws: fp8_linear_workspace_bytes() bytes of scratch.
 * saved == NULL: forward-only FP8 (inference, the paper's float8 dynamic activation +
 *   weight quantisation, PAPER.md:470-471 / 636, "same configurations as FP8
 *   training" PAPER.md:364-366): only the forward operands are cast (rowwise: row
 *   scales only; mxfp8: dim0 only) and `ws` must hold
 *   fp8_linear_infer_workspace_bytes() bytes.
 * ------------------------------------------------------------------------- */
size_t fp8_linear_saved_bytes(const fp8_linear_cfg_t* cfg, int64_t M, int64_t N, int64_t K);

/* Where one linear's FP8 operands live inside its `saved` and `ws` buffers (inspection: parity
 * tests byte-check exactly what fp8_linear_fwd / fp8_linear_bwd wrote; checkpoint tooling).  Fills
 * `out` with pointers into the caller's buffers (no device access, no launch); NULL entries are
 * operands the recipe does not have.  Forward-workspace entries hold the forward's operands
 * after fp8_linear_fwd until the next call using `ws` (the backward reuses it); backward entries
 * hold the backward's dY operands after fp8_linear_bwd.  Layouts (R-c17, operand plan §2):
 *   tensorwise: x_fwd = x_bwd = Xq [M,K], w_fwd = w_bwd = Wq [N,K], float[1] scales;
 *     dy_dx = dy_dw = Gq [M,N], float[1];
 *   rowwise (+_gw_hp): x_fwd [M,K] row-scaled (float[M]), w_fwd [N,K] row-scaled (float[N]),
 *     x_bwd [M,K] column-scaled (float[K]; NULL for gw_hp), w_bwd [N,K] column-scaled (float[K]),
 *     dy_dx [M,N] row-scaled (float[M]), dy_dw [M,N] column-scaled (float[N]; NULL for gw_hp);
 *   mxfp8: x_fwd/w_fwd/dy_dx dim0 codes in the input layout with blocked E8M0 [rows, cols/32];
 *     x_bwd [M,K], w_bwd [N,K], dy_dw [M,N] dim1 codes (blocks of 32 along the row index) in the
 *     input layout -- or transposed ([K,M], [K,N], [N,M]) when knob mx_transposed = 1
 *     (bwd_transposed) -- with blocked E8M0 [cols, rows/32].
 *   amax_fwd: tensorwise [amax X, amax W]; rowwise [X rows M | X cols K | W rows N | W cols K];
 *   amax_bwd: tensorwise [amax dY]; rowwise [dY rows M | dY cols N]; mxfp8: NULL (per-block amax
 *     is never stored). */
typedef struct {
  uint8_t* x_fwd; void* x_fwd_scale; uint8_t* w_fwd; void* w_fwd_scale;
  uint8_t* x_bwd; void* x_bwd_scale; uint8_t* w_bwd; void* w_bwd_scale;
  uint8_t* dy_dx; void* dy_dx_scale; uint8_t* dy_dw; void* dy_dw_scale;
  float* amax_fwd; float* amax_bwd;
  int bwd_transposed;
} fp8_linear_buffers_t;
fp8_status_t fp8_linear_buffers(const fp8_linear_cfg_t* cfg, int64_t M, int64_t N, int64_t K, void* saved,
                                void* ws, fp8_linear_buffers_t* out);
size_t fp8_linear_workspace_bytes(const fp8_linear_cfg_t* cfg, int64_t M, int64_t N, int64_t K);
size_t fp8_linear_infer_workspace_bytes(const fp8_linear_cfg_t* cfg, int64_t M, int64_t N, int64_t K);
fp8_status_t fp8_linear_fwd(const fp8_linear_cfg_t* cfg, fp8_hp_t x, fp8_hp_t w,
                            const fp8_tensor_t* w_fp8, void* y, void* saved,
                            void* ws, size_t ws_bytes, void* stream);

/* Forward with amax hand-over ("amax out of the critical path"; the
 * dynamic-quantisation overhead of PAPER.md:284-287):
 *   x_amax (nullable, device float[1], tensorwise only): amax(|X|) already known -- e.g. written
 *     by the epilogue of the GEMM that produced X -- so the X amax pass is skipped;
 *   y_amax (nullable, device float[1], any recipe): the GEMM epilogue writes amax(|Y|) of the
 *     stored (out_dtype-rounded) outputs, ready to be the next layer's x_amax.  It is zeroed on
 *     `stream` only after every cast has read x_amax, so x_amax and y_amax may share a buffer.
 * fp8_linear_fwd(...) == fp8_linear_fwd_ex(..., x_amax = NULL, ..., y_amax = NULL, ...). */
fp8_status_t fp8_linear_fwd_ex(const fp8_linear_cfg_t* cfg, fp8_hp_t x, const float* x_amax, fp8_hp_t w,
                               const fp8_tensor_t* w_fp8, void* y, float* y_amax, void* saved,
                               void* ws, size_t ws_bytes, void* stream);

/* Float8Linear backward: dX = dY W and dW = dY^T X (S:289-299 notation):
 *   tensorwise: dY one scale, reuse X/W scales; rowwise: dY per row for dX and
 *   per column for dW, W per column, X per column ("rows of the left
 *   operand, columns of the right"); mxfp8: dY blocks along N (dX) and along M
 *   (dW), W along N, X along M.
 * dy [M,N]; dx [M,K] and dw [N,K] out_dtype dense, either may be NULL.
 * x: the forward's input [M,K]; its shape gives K.  Its data is read only by
 *   FP8_RECIPE_ROWWISE_GW_HP, whose dW = dY^T X is a BF16 x BF16 tcgen05 GEMM
 *   (kind::f16, fp32 accumulate) on the high-precision dY and X (both must be BF16);
 *   for the other recipes x.ptr may be NULL.
 * `saved` must be the buffer the matching fp8_linear_fwd wrote.  If the forward
 * ran with a pre-cast weight (w_fp8), pass the same codes again (FSDP2 re-gathers
 * the weight for the backward); otherwise pass NULL. */
fp8_status_t fp8_linear_bwd(const fp8_linear_cfg_t* cfg, fp8_hp_t dy, fp8_hp_t x,
                            const void* saved, const fp8_tensor_t* w_fp8, void* dx, void* dw,
                            void* ws, size_t ws_bytes, void* stream);
/* Backward with amax hand-over: dy_amax (tensorwise only) skips the dY amax pass; dx_amax gets
 * amax(|dX|) from the dX GEMM epilogue (the previous layer's dy_amax).  May share a buffer. */
fp8_status_t fp8_linear_bwd_ex(const fp8_linear_cfg_t* cfg, fp8_hp_t dy, const float* dy_amax, fp8_hp_t x,
                               const void* saved, const fp8_tensor_t* w_fp8, void* dx, float* dx_amax,
                               void* dw, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Float8Linears sharing one input -- e.g. a Llama layer's wq / wk / wv (all read the attention
 * norm's output) and w1 / w3 (the MLP norm's output).  Each member is the Float8Linear of
 * fp8_linear_fwd / fp8_linear_bwd (Appendix A): X's scales depend on X alone
 * (tensorwise amax over X; rowwise per row / per column of X; MX blocks of X), so its amax and
 * FP8 copies are computed ONCE and read by every member's GEMMs (rowwise: X's and every W_i's row /
 * column amax by one launch and their FP8 copies by one cast launch; the backward likewise for every
 * dY_i; knob group_batch = 0 casts member by member).  Every output and every saved byte equals what
 * n separate fp8_linear_fwd / fp8_linear_bwd calls write.
 *   fwd: x [M,K]; w: HOST array of n weights [N_i, K] (fp32 or bf16 each); y: HOST array of n
 *     outputs [M, N_i] (out_dtype, dense); saved: HOST array of n buffers of
 *     fp8_linear_saved_bytes(cfg, M, N_i, K) bytes -- saved[0] holds X's backward operand,
 *     saved[i > 0] only W_i's; ws >= fp8_linear_shared_workspace_bytes(cfg, M, K, n, N) bytes (every
 *     member's forward W operand and backward dY operands side by side: the members' GEMMs -- Y_i in
 *     the forward, dX_i and dW_i in the backward -- run as ONE persistent launch per pass, up to 6
 *     problems per launch, so the small members (wk, wv) have no wave tail of their own).
 *   bwd: dy: HOST array of n [M, N_i]; x as for fp8_linear_bwd (data read by rowwise_gw_hp only);
 *     saved: the same array the forward wrote (all n, saved[0] first); dx / dw: HOST arrays of n
 *     outputs or NULL, entries may be NULL (dX_i is per member: summing the members' dX_i is the
 *     caller's -- autograd's -- job, as for separate linears); ws as for the forward (the same buffer
 *     may serve both passes).
 *   1 <= n <= FP8_SHARED_MAX.  No pre-cast weights (w_fp8) and no amax hand-over here.  All
 *   arguments are validated before the first launch.
 * ------------------------------------------------------------------------- */
#define FP8_SHARED_MAX 8
/* N: HOST int64[n], the members' output widths N_i.  0 for bad arguments. */
size_t fp8_linear_shared_workspace_bytes(const fp8_linear_cfg_t* cfg, int64_t M, int64_t K, int n, const int64_t* N);
fp8_status_t fp8_linear_fwd_shared(const fp8_linear_cfg_t* cfg, fp8_hp_t x, int n, const fp8_hp_t* w,
                                   void* const* y, void* const* saved, void* ws, size_t ws_bytes, void* stream);
fp8_status_t fp8_linear_bwd_shared(const fp8_linear_cfg_t* cfg, int n, const fp8_hp_t* dy, fp8_hp_t x,
                                   const void* const* saved, void* const* dx, void* const* dw, void* ws,
                                   size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * MoE scaled grouped GEMM ("scaled_grouped_mm: differentiable scaled
 * grouped GEMM for MoE FP8 training"; reading R-c22): the Float8Linear recipe applied
 * per expert to expert-sorted tokens, each pass ONE persistent tcgen05 launch.
 *   x [T,K] tokens sorted by expert; w [E*N, K] the E expert weights stacked (expert g
 *   = rows g*N..(g+1)*N-1, nn.Linear layout); dy [T,N]; y [T,N], dx [T,K], dw [E*N,K].
 *   offs: DEVICE int32[E+1], offs[0] = 0 <= offs[1] <= ... <= offs[E] = T, every entry
 *   a multiple of 128 (MoE token groups padded to 128 rows); expert g owns token rows
 *   [offs[g], offs[g+1]); empty experts allowed (dW_g = 0).  The offsets are validated
 *   on the device: a violation makes the GEMM compute no tile of that problem and sets the
 *   process fault word, reported as FP8_EINVAL by fp8_check_async_error (and by the next
 *   grouped call) -- the call never reads them on the host, so it never synchronises.
 *   Recipes: tensorwise (one scale per X, W, dY) or rowwise (per token row, per expert
 *   weight row / column, per (expert, column) over the expert's tokens for dW).
 *   T, N multiples of 128; K multiple of 16; 1 <= E <= 256.
 *   saved: fp8_grouped_saved_bytes(); ws: fp8_grouped_workspace_bytes() bytes.
 *   x in fp8_grouped_linear_bwd gives K only (ptr may be NULL).
 * ------------------------------------------------------------------------- */
size_t fp8_grouped_saved_bytes(const fp8_linear_cfg_t* cfg, int64_t T, int64_t E, int64_t N, int64_t K);
size_t fp8_grouped_workspace_bytes(const fp8_linear_cfg_t* cfg, int64_t T, int64_t E, int64_t N, int64_t K);
fp8_status_t fp8_grouped_linear_fwd(const fp8_linear_cfg_t* cfg, fp8_hp_t x, fp8_hp_t w, int64_t E,
                                    const int32_t* offs, void* y, void* saved, void* ws,
                                    size_t ws_bytes, void* stream);
fp8_status_t fp8_grouped_linear_bwd(const fp8_linear_cfg_t* cfg, fp8_hp_t dy, fp8_hp_t x, int64_t E,
                                    const int32_t* offs, const void* saved, void* dx, void* dw,
                                    void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * FSDP2-style FP8 weight all-gather (PAPER.md:596 enable_fp8_all_gather;
 * reading R-c18): per rank, amax of the local shard -> NCCL all-reduce MAX ->
 * s = RN32(fmax / max(amax, eps)) -> cast the shard into slot `rank` of
 * w_full -> NCCL all-gather of the bytes.  The result is bit-identical on
 * every rank and equal to the unsharded tensorwise cast.
 *   w_shard  [rows_local, cols] high precision (this rank's rows)
 *   w_full   [nranks * rows_local, cols] u8 codes (device)
 *   scale_out float[1], amax_out float[1] (device; the global amax)
 *   ws: fp8_fsdp_workspace_bytes() bytes.
 * ------------------------------------------------------------------------- */
typedef struct fp8_comm_s* fp8_comm_t;
/* Host: fill id[128] on one rank (ncclGetUniqueId); broadcast it yourself. */
fp8_status_t fp8_comm_get_unique_id(uint8_t id[128]);
/* Host, collective over nranks processes; binds the communicator to the
 * current CUDA device. */
fp8_status_t fp8_comm_init(fp8_comm_t* comm, const uint8_t id[128], int nranks, int rank);
fp8_status_t fp8_comm_destroy(fp8_comm_t comm);
/* Communicator health: FP8_ENCCL if NCCL reports an asynchronous error on it (ncclCommGetAsyncError:
 * a peer failed, a timed-out or aborted operation), or the pending device fault (fp8_check_async_error).
 * The FSDP entry points run the same check before enqueuing work. */
fp8_status_t fp8_comm_check(fp8_comm_t comm);
size_t fp8_fsdp_workspace_bytes(fp8_hp_t w_shard);
fp8_status_t fp8_fsdp_allgather(fp8_comm_t comm, fp8_hp_t w_shard, fp8_format_t fmt,
                                uint8_t* w_full, float* scale_out, float* amax_out,
                                void* ws, size_t ws_bytes, void* stream);
/* Precomputed global amax for all of a model's FP8-gathered weights at once (the
 * torchtitan-style precompute after the optimizer step): one
 * fp8_amax_multi launch over this rank's n shards + ONE ncclAllReduce(MAX) of the n
 * amaxes.  amax_out: device float[n] (the global amaxes), 1 <= n <= 48. */
fp8_status_t fp8_fsdp_precompute_amax(fp8_comm_t comm, const fp8_hp_t* w_shards, int n,
                                      float* amax_out, void* stream);
/* As fp8_fsdp_allgather, but with amax_in = the global amax from
 * fp8_fsdp_precompute_amax (device float[1]): no amax pass and no all-reduce, only
 * cast-into-slot + all-gather.  amax_in NULL = fp8_fsdp_allgather. */
fp8_status_t fp8_fsdp_allgather_ex(fp8_comm_t comm, fp8_hp_t w_shard, fp8_format_t fmt,
                                   const float* amax_in, uint8_t* w_full, float* scale_out,
                                   float* amax_out, void* ws, size_t ws_bytes, void* stream);

/* MXFP8 FSDP weight all-gather (MX formats for training, PAPER.md:735;
 * FSDP gathers in low precision).  E8M0 block scales are shard-local -- a
 * 32-block never crosses a shard boundary when rows_local % 128 == 0 -- so there is no amax
 * exchange: rank r casts its shard [rows_local, cols] straight into slot r of
 *   out->q       [nranks*rows_local, cols] u8  dim0 codes (blocks of 32 along cols = K: the
 *                                               forward GEMM's W operand)
 *   out->scale   E8M0 blocked [N, K/32]         (N = nranks*rows_local, K = cols)
 *   out->q_t     [N, K] u8                      dim1 codes (blocks of 32 along rows = N: the dX
 *                                               GEMM's W operand), row-major MX32_RM layout
 *   out->scale_t E8M0 blocked [K, N/32]
 * then one NCCL group all-gathers the four buffers, and the dim1 scales (gathered rank-major
 * into `ws`) are re-tiled into the blocked layout of the full matrix.  The result is
 * bit-identical on every rank and equal to fp8_cast_scaled(W, MX32_RM) of the unsharded W.
 * out->gran must be FP8_GRAN_MX32_RM; out->q_t / out->scale_t may both be NULL (forward-only
 * gather: dim0 only, no workspace).  rows_local, cols: multiples of 128.  `out` may be passed
 * as w_fp8 to fp8_linear_fwd / fp8_linear_bwd with the mxfp8 recipe.
 * ws: fp8_fsdp_mx_workspace_bytes(w_shard, nranks) bytes (device). */
size_t fp8_fsdp_mx_workspace_bytes(fp8_hp_t w_shard, int nranks);
fp8_status_t fp8_fsdp_allgather_mx(fp8_comm_t comm, fp8_hp_t w_shard, fp8_mx_round_t mx_round,
                                   fp8_tensor_t* out, void* ws, size_t ws_bytes, void* stream);
/* The re-tiling step of fp8_fsdp_allgather_mx, exported for composition: rank_major holds
 * nranks consecutive E8M0 blocked buffers, buffer p = the dim1 scales of shard p
 * ([cols, rows_local/32] blocked); out gets the blocked [cols, nranks*rows_local/32] buffer.
 * rows_local, cols multiples of 128; pointers 16-byte aligned; async on `stream`. */
fp8_status_t fp8_mx_scales_unshard(const uint8_t* rank_major, int nranks, int64_t rows_local,
                                   int64_t cols, uint8_t* out, void* stream);

/* ---------------------------------------------------------------------------
 * Fused FP8 FSDP all-gather over NVLink peer memory (the B200-native form of the
 * tensorwise enable_fp8_all_gather of PAPER.md:596, reading R-c18).  The cast kernel
 * stores each rank's FP8 codes straight into slot `rank` of EVERY rank's gather buffer
 * (CUDA-IPC peer pointers over NVLink / NVSwitch): the all-gather's data movement is
 * the cast's own output stream, with no NCCL kernel and no local round trip of the
 * codes.  The global amax is exchanged through per-rank signal slots in the same
 * windows (release/acquire at system scope), which also serves as the barrier that
 * keeps a fast rank from overwriting a buffer a slow rank is still reading.
 * Result: bit-identical to fp8_fsdp_allgather (and to the unsharded tensorwise cast).
 * ------------------------------------------------------------------------- */
typedef struct fp8_p2p_s* fp8_p2p_t;
/* Host, collective over the communicator's ranks: allocate this rank's window (a
 * gather buffer of `bytes` + a signal block, zeroed), exchange CUDA IPC handles over
 * NCCL, open every peer's window (needs peer access: NVLink / NVSwitch).  One window
 * per concurrently live gathered weight; bytes >= nranks * rows_local * cols. */
fp8_status_t fp8_p2p_create(fp8_comm_t comm, size_t bytes, fp8_p2p_t* win);
/* The two halves of fp8_p2p_create for callers that exchange the handles themselves (e.g. over
 * a torch gloo group): fp8_p2p_alloc allocates and zeroes this rank's window and returns its
 * 64-byte CUDA IPC handle; after every rank's handle is known (handles = nranks x 64 bytes in rank
 * order), fp8_p2p_open maps the peers.  The caller must then barrier (no rank may signal into a
 * peer before that peer's fp8_p2p_alloc has returned). */
fp8_status_t fp8_p2p_alloc(size_t bytes, int nranks, int rank, fp8_p2p_t* win, uint8_t handle[64]);
fp8_status_t fp8_p2p_open(fp8_p2p_t win, const uint8_t* handles);
/* Test / single-GPU form: nranks windows on the current device, wins[r] acting as rank
 * r, all mapped to each other (plain device pointers).  Drive it with
 * fp8_fsdp_allgather_p2p_local (one stream); per-rank calls on separate streams would
 * rely on those streams running concurrently, which CUDA does not guarantee. */
fp8_status_t fp8_p2p_create_local(int nranks, size_t bytes, fp8_p2p_t* wins);
/* Device pointer of this rank's gather buffer: the codes [nranks*rows_local, cols] u8
 * after fp8_fsdp_allgather_p2p (valid in stream order after the call). */
void* fp8_p2p_buffer(fp8_p2p_t win);
fp8_status_t fp8_p2p_destroy(fp8_p2p_t win);
/* Per rank, on `stream` (every rank calls it for the same weight in the same order):
 *   amax(W_r) (skipped if amax_in, a device float[1] global amax, e.g. from
 *   fp8_fsdp_precompute_amax) -> signal it into every peer's slot r -> wait for all
 *   P slots, s = RN32(fmax / max(max_p amax_p, eps)) -> scale_out (device float[1]),
 *   amax_out (device float[1], the global amax; also the accumulator when amax_in is
 *   NULL) -> cast W_r pushing codes to every peer -> wait until every rank's pushes
 *   into this buffer are visible.  Spins carry a 10 s watchdog (kernel trap ->
 *   FP8_ECUDA at the next sync) instead of hanging.  w_shard rows/cols multiples of 16. */
fp8_status_t fp8_fsdp_allgather_p2p(fp8_p2p_t win, fp8_hp_t w_shard, fp8_format_t fmt,
                                    const float* amax_in, float* scale_out, float* amax_out,
                                    void* stream);
/* Single-process form for a fp8_p2p_create_local group: rank r's call with shard w[r] for every
 * r, issued phase by phase on ONE stream (all signals, then all scale waits, then all casts,
 * then all completion waits), so the ranks' spins never wait on work queued behind them.
 * amax_in / amax_out may be NULL arrays (amax_out[r] is needed when amax_in is NULL). */
fp8_status_t fp8_fsdp_allgather_p2p_local(fp8_p2p_t* wins, int nranks, const fp8_hp_t* w_shards,
                                          fp8_format_t fmt, const float* const* amax_in,
                                          float* const* scale_out, float* const* amax_out,
                                          void* stream);
/* Async-TP FP8 linear forward ("float8 training with async
 * tensor parallelism"): sequence-parallel activations X_r [M_local, K] (rank r's tokens) are
 * all-gathered in FP8 and multiplied by this rank's column shard of the weight W_r [N_local, K],
 *   y [nranks*M_local, N_local] = X_full W_r^T,
 * with the gather and the GEMM overlapped inside ONE GEMM launch: each rank's cast kernel pushes
 * its codes (tensorwise, one global scale from the same amax signal slots as the FSDP gather)
 * into slot r of every window and publishes done[r]; the GEMM's TMA producer waits for done[c]
 * before loading the rows of chunk c, computing its own chunk first.  The window (from
 * fp8_p2p_create) must hold nranks*M_local*K bytes; M_local % 256 == 0; cfg->recipe
 * tensorwise; y and ws 256-byte aligned; ws: fp8_tp_workspace_bytes(N_local, K) bytes. */
size_t fp8_tp_workspace_bytes(int64_t n_local, int64_t K);
fp8_status_t fp8_tp_allgather_linear_fwd(fp8_p2p_t win, const fp8_linear_cfg_t* cfg, fp8_hp_t x_shard,
                                         fp8_hp_t w, void* y, void* ws, size_t ws_bytes, void* stream);
/* FSDP backward with the dW reduce-scatter fused into the dW GEMM (the "GEMM -> reduce-scatter"
 * pattern; FSDP2 reduce-scatters weight gradients to their dim-0 shards): as fp8_linear_bwd, but
 * every dW tile is stored by the GEMM epilogue straight into the staging buffer of the rank that
 * owns its rows (rs_win: a window of >= nranks * (N/nranks) * K * 2 bytes from fp8_p2p_create, one
 * per concurrently reduced gradient), and this rank then sums its nranks slots in rank order
 * (fp32, one bf16 rounding) into dw_shard [N/nranks, K] bf16.  dx is computed locally as usual.
 * Every rank calls it in the same order; N % (256 * nranks) == 0; cfg->out_dtype BF16.  A
 * cross-rank barrier on rs_win at entry keeps a fast rank from overwriting a slot a slow rank is
 * still summing.  Result == the bf16 sum of the ranks' fp8_linear_bwd dW rows (bit-exact). */
fp8_status_t fp8_linear_bwd_rs(const fp8_linear_cfg_t* cfg, fp8_hp_t dy, fp8_hp_t x, const void* saved,
                               const fp8_tensor_t* w_fp8, void* dx, fp8_p2p_t rs_win, int nranks,
                               void* dw_shard, void* ws, size_t ws_bytes, void* stream);
/* Async-TP FP8 linear backward (pairs with fp8_tp_allgather_linear_fwd; "GEMM -> reduce-scatter"):
 *   dy [M, N_local] (this rank's output columns, all M tokens), tensorwise local scale;
 *   dw [N_local, K] bf16 = dY^T X_full using the FP8 X codes the forward gathered into `win`
 *     (call before the next forward on `win`) and its global X scale (fwd_ws = the forward's ws);
 *   dx_shard [M/nranks, K] bf16 = sum over ranks of (dY_r W_r)[this rank's token rows]: the dX
 *     GEMM's epilogue stores each tile into the staging slot of the rank owning its rows (rs_win,
 *     >= M * K * 2 bytes), which sums its nranks slots in rank order (fp32, one bf16 rounding).
 * dX and dW share one persistent launch.  M % (256 * nranks) == 0; ws:
 * fp8_tp_bwd_workspace_bytes(M, N_local) bytes (256-byte aligned). */
size_t fp8_tp_bwd_workspace_bytes(int64_t M, int64_t n_local);
fp8_status_t fp8_tp_linear_bwd(fp8_p2p_t win, const void* fwd_ws, fp8_p2p_t rs_win, const fp8_linear_cfg_t* cfg,
                               fp8_hp_t dy, int64_t K, void* dx_shard, void* dw, void* ws, size_t ws_bytes,
                               void* stream);
/* Single-process form for a fp8_p2p_create_local group (phase by phase on one stream). */
fp8_status_t fp8_tp_allgather_linear_fwd_local(fp8_p2p_t* wins, int nranks, const fp8_linear_cfg_t* cfg,
                                               const fp8_hp_t* x_shards, const fp8_hp_t* w, void* const* y,
                                               void* const* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Helpers
 * ------------------------------------------------------------------------- */
int fp8_abi_version(void);
/* Asynchronous device faults.  Kernels that wait on other ranks (the P2P FSDP gather, the fused
 * reduce-scatter, async-TP) give up after the watchdog (knob watchdog_ms, default 30 s) instead of
 * trapping -- a trap would poison the CUDA context -- and record a fault code in a process-wide word of
 * pinned, device-mapped host memory; grouped GEMMs record invalid device offsets the same way.  The
 * outputs of the call that faulted are invalid.  fp8_check_async_error() returns FP8_OK or the recorded
 * fault (FP8_ECUDA / FP8_EINVAL, with fp8_last_error() naming the rank / chunk / epoch) and clears it;
 * every P2P, async-TP, fused reduce-scatter, grouped and FSDP entry point performs the same check first.
 * Like any asynchronous CUDA error, a fault becomes visible only after the faulting kernel ran. */
fp8_status_t fp8_check_async_error(void);
/* Thread-local message describing the last non-OK status of this thread. */
const char* fp8_last_error(void);
/* Number of kernels this library has launched in the calling process (all
 * threads); for launch accounting in benchmarks. */
uint64_t fp8_launch_count(void);

/* Kernel-variant knobs (host-side, process-wide, thread-safe).  The library never reads the
 * process environment; every variant other than the product default is selected explicitly:
 *   amax_tile_tma (1) | cast_grid (0 = uncapped) | amax_blocks_per_sm (8) | amax_loads (8) |
 *   mx_cast_tma (1) | gemm_cta_group (2) | gemm_debug (0) | gemm_sched (1 = dynamic) |
 *   mx_sf_split (1) | gemm_raster (-1 = per problem) | mx_n192 (0) | gemm_stages (3) |
 *   gemm_epi (0 = by K) | mx_transposed (0; forward and backward of one linear must agree) |
 *   tw_dual (1) | gemm_kserp (1: odd waves of GEMM tiles walk K backwards) |
 *   gemm_n512 (2 = 256 x 512 tiles for plain FP8 launches whose problems all have N % 512 == 0 and
 *   K >= 8192; 1 = whenever N % 512 == 0; 0 = never) |
 *   gemm_l2pf (0 = off; d > 0: the GEMM producer prefetches operand boxes d stages ahead into L2) |
 *   mx_cast_occ3 (0) | amax_bulk (1: tensorwise amax of contiguous tensors by 1-D bulk copies; 0: register streaming) |
 *   amax_rc (1: row / column amax by the multi-tensor warp-specialised kernel; 0: amax_tile_tma's choice) |
 *   amax_rc_debug (0; A/B probes only) | group_batch (1: a rowwise shared-input group's amax and cast launches
 *   batched over X and every W_i, and over every dY_i; 0: per member) |
 *   mx_cast_ws (0; 1 = bf16 MX casts with row-major dim1 copies by the warp-specialised kernel) | mx_cast_debug (0) |
 *   gemm_st_ef (0: 1 = GEMM bf16 outputs stored with an L2 evict-first hint) | wait_sleep (0; bit mask: barrier waits
 *   sleep with a suspend-time hint -- 1 amax_rc / MX casts, 2 GEMM epilogue, 4 GEMM producer, 8 GEMM MMA) |
 *   gemm_l2hint (0; A/B: 1 = GEMM A operand loads evict_last, 2 = + B evict_first) |
 *   gemm_afill (0; 1 = 256 x 512 tiles issue both halves' MMAs per K step with A held in the collector) |
 *   mx_cast_tstore (1: the MX ring cast writes its dim0 / row-major dim1 codes by TMA tensor stores; 0: st.global) |
 *   cast_rc_tma (1: rowwise casts of launches up to 12288 tiles by the persistent TMA kernel with TMA stores;
 *   2: always; 0: never) |
 *   cast_rc_wide (0; A/B) | gemm_epi_tma (0; 1 = 256-wide GEMM tiles write bf16 outputs by TMA stores) |
 *   watchdog_ms (30000; 0 = peer waits never give up)
 *   -- defaults in parentheses.
 * A knob changes launches enqueued after the call.  Unknown name or out-of-range value:
 * FP8_EINVAL, nothing changed.  fp8_reset_knobs restores every default. */
fp8_status_t fp8_set_knob(const char* name, int value);
fp8_status_t fp8_get_knob(const char* name, int* value);
void fp8_reset_knobs(void);

/* Per-launch device timing for benchmarks.  While enabled, every kernel this library
 * launches is bracketed by two CUDA events recorded on its own stream.
 * fp8_profile_collect() waits for the recorded events, writes up to max_n records
 * (kind, duration in ms) in launch order and clears the list; returns the number of
 * records written (or -1 on a CUDA error).  Kinds: 0 amax, 1 cast, 2 mx_cast,
 * 3 transpose_u8 (and the MX scale re-tiling), 4 gemm (FP8), 5 gemm (MXFP8), 6 gemm (BF16,
 * rowwise_gw_hp dW), 7 P2P gather signal / wait kernels. */
void fp8_profile_enable(int on);
int fp8_profile_collect(int* kinds, float* ms, int max_n);

#ifdef __cplusplus
}
#endif
#endif /* FP8TRAIN_H_ */
