/*
 * fpsa.h -- C ABI of the B200-native FPSAttention hot path (libfpsa.so).
 *
 * Drop-in boundary for the reference package fp8sta (arXiv 2506.04648,
 * /root/reference/pkg/src/fp8sta).  The reference has no FFI: its boundary
 * is the Python surface re-exported in fp8sta/__init__.py:10-48.  Each entry
 * point below replaces one reference function (cited per function); the
 * Python package paper_2506_04648_b200 binds them with ctypes and mirrors the
 * reference names, argument meaning and exceptions on top.
 *
 * Conventions
 *   - plain pointers and sizes, no torch types; every call returns an int
 *     status (FPSA_OK == 0, see fpsa_status);
 *   - device buffers are caller-owned; device calls are asynchronous on the
 *     given cudaStream_t (passed as void*; NULL = legacy default stream) and
 *     allocate nothing (workspaces are caller-provided);
 *   - no global mutable state except a per-process table of driver entry
 *     points, initialised once and thread-safe;
 *   - token grids are (t, h, w) with w fastest (fp8sta/grid.py:1-8);
 *   - "tile-major padded" code layout: for head h, tile u, local row r,
 *     row index (h*M + u)*tile_pitch + r of a [rows][d] uint8 matrix, rows
 *     r in [tile_volume, tile_pitch) zero.  tile_pitch == tile_volume gives
 *     exactly the reference's tile-contiguous layout (fp8sta/grid.py:132-154).
 */
#ifndef FPSA_H_
#define FPSA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FPSA_OK = 0,
  FPSA_EINVAL = 1,        /* bad argument (reference: ValueError) */
  FPSA_EINDIVISIBLE = 2,  /* tile does not divide grid (grid.py:95-99, ValueError) */
  FPSA_ENONFINITE = 3,    /* non-finite input (quantize.py:105-106, attention.py:53-54) */
  FPSA_ECUDA = 4,         /* CUDA runtime / driver error */
  FPSA_EUNSUPPORTED = 5,  /* valid request this build does not implement (e.g. d not in {64,128}) */
  FPSA_ERANGE = 6,        /* index out of range (reference: IndexError) */
  FPSA_ECAPACITY = 7      /* caller buffer too small */
} fpsa_status;

typedef enum { FPSA_F32 = 0, FPSA_BF16 = 1, FPSA_F16 = 2, FPSA_F64 = 3 } fpsa_dtype;
typedef enum { FPSA_E4M3 = 0, FPSA_E5M2 = 1 } fpsa_fmt;
typedef enum { FPSA_ORDER_TILE = 0, FPSA_ORDER_NATURAL = 1 } fpsa_order;
/* Softmax-weight semantics of fpsa_attn_fwd: one-pass (unnormalised weights re-quantised per key block,
 * the fast path) or normalised (the reference's exact P = e4m3(448 * p), attention.py:133-145). */
typedef enum { FPSA_P_ONEPASS = 0, FPSA_P_NORMALIZED = 1 } fpsa_p_mode;

typedef struct {
  int32_t t, h, w;
} fpsa_dims3;

/* Human-readable text of the last error on this thread ("" if none). */
const char* fpsa_last_error(void);
/* ABI version, major*10000 + minor*100 + patch. */
int fpsa_version(void);

/* ---------------------------------------------------------------- host layout */

/* Tiles per axis of grid/tile; FPSA_EINDIVISIBLE with the reference message
 * text in fpsa_last_error().  Replaces build_tile_map (fp8sta/grid.py:91-109). */
int fpsa_tile_grid(fpsa_dims3 grid, fpsa_dims3 tile, fpsa_dims3* tile_dims);

/* Gather permutation to tile-major order, perm[L].  Replaces
 * tile_contiguous_order (fp8sta/grid.py:132-154). */
int fpsa_tile_perm(fpsa_dims3 grid, fpsa_dims3 tile, int64_t* perm);

/* Number of admissible (query tile, key tile) pairs of a window.  With
 * fpsa_window_csr replaces build_block_mask / BlockMask.allowed /
 * allowed_counts / density (fp8sta/sparsity.py:48-75, :112-144). */
int fpsa_window_nnz(fpsa_dims3 tile_dims, fpsa_dims3 window, int64_t* nnz);

/* CSR of ascending admissible key tiles per query tile:
 * offs[M+1], ids[nnz] (capacity `cap`). */
int fpsa_window_csr(fpsa_dims3 tile_dims, fpsa_dims3 window, int32_t* offs, int32_t* ids, int64_t cap,
                    int64_t* nnz);

/* Regime index (0 early, 1 mid, 2 late) of 1-based step t.  Replaces
 * ScheduleConfig.regime_of / params_at (fp8sta/schedule.py:41-50, :71-73). */
int fpsa_regime_of(int32_t t, int32_t total_steps, double alpha1, double alpha2, int32_t* regime);

/* ---------------------------------------------------------------- device kernels */

/* Per-3D-tile FP8 quantisation of q or k for `heads` heads in one pass:
 * read x (dtype, element (token, head, c) at x + token*token_stride +
 * head*head_stride + c, tokens in `in_order`), gather to tile-major order,
 * per-tile amax, f64 scale = amax/max_value (1.0 for an all-zero tile), e4m3 /
 * e5m2 codes bit-identical to the reference (round-to-nearest-even of the f64
 * quotient).  codes: tile-major padded [heads*M*tile_pitch][d];
 * scales: f64 [heads*M].  err_flag (device int32, may be NULL) gets bit 0 set
 * on non-finite input.  Replaces quantize_qk_tilewise (fp8sta/quantize.py:111-124)
 * together with tile_contiguous_order and fp8.encode (fp8.py:153-188). */
int fpsa_quantize_qk(const void* x, int dtype, int64_t token_stride, int64_t head_stride, int32_t heads,
                     fpsa_dims3 grid, fpsa_dims3 tile, int32_t d, int32_t tile_pitch, int in_order, int fmt,
                     uint8_t* codes, double* scales, int32_t* err_flag, void* stream);

/* Per-channel FP8 quantisation of v: column amax over all L tokens of each
 * head, f64 scale per (head, channel), codes in the same tile-major padded
 * layout as fpsa_quantize_qk.  workspace: device, >= heads*d*8 bytes.
 *
 * Both quantisers accept any head dim d >= 1 and f32 / bf16 / f64 input
 * (the reference quantises any L x d float64 matrix): d in {64, 128} with
 * f32 / bf16 runs the fast kernels; f64 or other d runs general kernels
 * that take every element through the exact f64 path (f64 maxima).
 * Replaces quantize_v_channelwise (fp8sta/quantize.py:127-134). */
int fpsa_quantize_v(const void* x, int dtype, int64_t token_stride, int64_t head_stride, int32_t heads,
                    fpsa_dims3 grid, fpsa_dims3 tile, int32_t d, int32_t tile_pitch, int in_order, int fmt,
                    uint8_t* codes, double* scales, void* workspace, int32_t* err_flag, void* stream);

/* Device workspace bytes of fpsa_quantize_qkv / fpsa_quantize_qkv_amax
 * ((2*heads*d + heads + 1) * 4: v channel maxima (8-byte on the general
 * path) plus spare words; zeroed by the call). */
int fpsa_quantize_workspace_bytes(int32_t heads, int32_t d, int64_t* bytes);

/* Fused form of fpsa_quantize_qk(q) + fpsa_quantize_qk(k) + fpsa_quantize_v(v)
 * for three tensors with the same dtype and strides, bit-identical to the
 * separate calls: one channel-amax pass over v, then a single persistent
 * TMA-fed launch over all q, k and v tiles (bf16, d = 128, tile volume <= 256;
 * otherwise one grid over all tiles).  workspace: device,
 * >= fpsa_quantize_workspace_bytes(heads, d). */
int fpsa_quantize_qkv(const void* q, const void* k, const void* v, int dtype, int64_t token_stride,
                      int64_t head_stride, int32_t heads, fpsa_dims3 grid, fpsa_dims3 tile, int32_t d,
                      int32_t tile_pitch, int in_order, int fmt, uint8_t* q_codes, uint8_t* k_codes,
                      uint8_t* v_codes, double* q_scales, double* k_scales, double* v_scales, void* workspace,
                      int32_t* err_flag, void* stream);

/* fpsa_quantize_qkv with the absolute maxima supplied by the producer of q, k, v
 * (the upstream-fusion hook, Alg. 1 steps 2-3: a QKV-projection
 * epilogue reduces |x| while it writes): q_tile_amax / k_tile_amax f32
 * [heads*M] (tile order), v_channel_amax f32 [heads*d]; any may be NULL
 * (computed here).  They must equal max|x| over the tile / channel, so the
 * codes and scales stay those of the reference.  With v_channel_amax the
 * channel-amax pass (an extra read of v) disappears; the tile maxima are
 * reduced from the tile in shared memory anyway. */
int fpsa_quantize_qkv_amax(const void* q, const void* k, const void* v, int dtype, int64_t token_stride,
                           int64_t head_stride, int32_t heads, fpsa_dims3 grid, fpsa_dims3 tile, int32_t d,
                           int32_t tile_pitch, int in_order, int fmt, const float* q_tile_amax,
                           const float* k_tile_amax, const float* v_channel_amax, uint8_t* q_codes,
                           uint8_t* k_codes, uint8_t* v_codes, double* q_scales, double* k_scales, double* v_scales,
                           void* workspace, int32_t* err_flag, void* stream);

/* Element codec.  fpsa_encode: codes[i] = RNE(x[i]) (scale == NULL) or
 * RNE(x[i] / scale[i]) with the quotient in f64 (scale: device f64 [n]),
 * onto e4m3 / e5m2, saturating finite magnitudes, sign kept on zero;
 * x dtype f32 / bf16 / f64 (an unscaled f32 is rounded as f32, everything else
 * through f64).  err_flag (device int32): bit 0 NaN input, bit 1 infinity in
 * a format without one (E5M2 infinities get the inf code).  Replaces
 * fp8.encode (fp8sta/fp8.py:153-188) and the division of quantize_dequantize
 * (:219-234). */
int fpsa_encode(const void* x, int dtype, const double* scale, int64_t n, int fmt, uint8_t* codes, int32_t* err_flag,
                void* stream);

/* fpsa_decode: out[i] = value(codes[i]) (* scale[i] in f64 when scale != NULL),
 * out dtype f32 / f64; a NaN code pattern sets err_flag bit 0.  Replaces
 * fp8.decode (fp8.py:191-205), QuantizedTensor.dequantize /
 * dequantize_tensor (quantize.py:95-98, :183-185) and the reconstruction of
 * quantize_dequantize. */
int fpsa_decode(const uint8_t* codes, int64_t n, int fmt, const double* scale, void* out, int out_dtype,
                int32_t* err_flag, void* stream);

/* Work list for fpsa_attn_fwd: one entry per (head, query tile, 128-row
 * query block), tiles with the most key tiles first within each head, the
 * query blocks of a tile adjacent (they stream the same K/V from L2).
 * Host-side; n_items returns the count, items (capacity `cap`, 3 int32 each:
 * head, tile, query block). */
int fpsa_attn_worklist(int32_t heads, fpsa_dims3 tile_dims, int32_t tile_volume, const int32_t* offs_host,
                       int32_t* items, int64_t cap, int64_t* n_items);

/* Bytes of device workspace fpsa_attn_fwd needs for n_items work items (the
 * list of items recomputed in exact mode, see below). */
int fpsa_attn_workspace_bytes(int32_t n_items, int64_t* bytes);

/* Sliding-tile sparse FP8 attention forward over quantised codes.
 * Persistent kernel over the work list; items whose one-pass softmax may have
 * saturated e4m3 (a logit more than tau_log2 above the first key block's row
 * max) are recomputed by a second, exact-max launch on the same stream.
 *   q/k/v codes: tile-major padded (fpsa_quantize_*), tile_pitch a multiple of 128
 *   q/k scales: f64 [heads*M]; v scales f64 [heads*d]
 *   offs/ids: device CSR from fpsa_window_csr; items/n_items: device work list
 *   softmax_scale > 0 (the reference default is f32(1/sqrt(d)))
 *   out: element (token, head, c) at out + token*out_token_stride +
 *        head*out_head_stride + c, tokens in out_order, dtype out_dtype
 *   tau_log2: headroom of the one-pass softmax above the first block's row max (0..8)
 *   p_mode: FPSA_P_ONEPASS, or FPSA_P_NORMALIZED: three passes per item (exact row max, f64 row sum,
 *           then P = e4m3(448 * exp(s - m) / f32(l)) with a correctly rounded exp) and
 *           out = O * f32(v_scale / 448): the reference's arithmetic step for step; f32 output only,
 *           no redo launch (tau_log2 unused)
 *   workspace: device, >= fpsa_attn_workspace_bytes(n_items); word 0 = number of
 *              items recomputed exactly by this call (readable after the stream syncs)
 * Replaces fp8_sparse_forward / _engine (fp8sta/attention.py:91-149, :179-208). */
int fpsa_attn_fwd(const uint8_t* q_codes, const uint8_t* k_codes, const uint8_t* v_codes, const double* q_scales,
                  const double* k_scales, const double* v_scales, int32_t heads, fpsa_dims3 grid, fpsa_dims3 tile,
                  int32_t d, int32_t tile_pitch, const int32_t* offs, const int32_t* ids, const int32_t* items,
                  int32_t n_items, float softmax_scale, int fmt, float tau_log2, int p_mode, void* out, int out_dtype,
                  int64_t out_token_stride, int64_t out_head_stride, int out_order, void* workspace,
                  int64_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------- passthrough (full precision)
 * The reference's passthrough branch / sparse_reference (fp8sta/attention.py:152-154,
 * :165-176, :192-194): the same sliding-tile sparse attention without FP8
 * quantisation, on bf16 operands with f32 softmax and accumulation. */

/* Gather [tokens, heads, d] (f32 or bf16, tokens in in_order, element (t, h, c)
 * at x + t*token_stride + h*head_stride + c) into the tile-major padded bf16
 * layout [heads][M][tile_pitch][d] the passthrough kernel reads; rows
 * tv..tile_pitch-1 of every tile are written as zero.  f32 is rounded to
 * nearest even.  Replaces AttentionInputs' tile-contiguous f32 copies
 * (fp8sta/attention.py:36-61) plus tile_contiguous_order (grid.py:132-154). */
int fpsa_tile_gather_bf16(const void* x, int dtype, int64_t token_stride, int64_t head_stride, int32_t heads,
                          fpsa_dims3 grid, fpsa_dims3 tile, int32_t d, int32_t tile_pitch, int in_order, void* out,
                          void* stream);

/* Passthrough attention over fpsa_tile_gather_bf16 buffers: for each query
 * row, softmax(scale * q k^T) v over the keys of its window tiles, with the
 * same work list, CSR, workspace, output layout and exact-max redo as
 * fpsa_attn_fwd (the redo is needed only when a logit exceeds the first key
 * block's row max by more than 127 / log2 e). */
int fpsa_attn_bf16_fwd(const void* q_tiles, const void* k_tiles, const void* v_tiles, int32_t heads,
                       fpsa_dims3 grid, fpsa_dims3 tile, int32_t d, int32_t tile_pitch, const int32_t* offs,
                       const int32_t* ids, const int32_t* items, int32_t n_items, float softmax_scale, void* out,
                       int out_dtype, int64_t out_token_stride, int64_t out_head_stride, int out_order,
                       void* workspace, int64_t workspace_bytes, void* stream);

/* Per-head fidelity sums of an approximation against a reference, both
 * [tokens, heads, d] with the same strides (f32 or bf16):
 * out (device, f64 [heads][6]) = sum(r a), sum(r r), sum(a a), sum((r-a)^2),
 * max|r|, max|a|.  The inputs of cosine_similarity / mse / snr_db
 * (fp8sta/metrics.py:41-88); the host finishes them. */
int fpsa_fidelity(const void* ref, int ref_dtype, const void* approx, int approx_dtype, int64_t tokens,
                  int32_t heads, int32_t d, int64_t token_stride, int64_t head_stride, double* out, void* stream);

/* Strided 2D copy (cudaMemcpy2DAsync, direction from the pointers): `rows`
 * rows of `width` bytes, row r from src + r*src_pitch to dst + r*dst_pitch.
 * Used by the streamed host path to move a run of heads of every token
 * between a pinned host [tokens, heads, d] array and a device
 * [tokens, chunk, d] buffer (the reference copies its inputs into f32
 * contiguous arrays, fp8sta/attention.py:50-57). */
int fpsa_copy2d(void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch, int64_t width, int64_t rows,
                void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FPSA_H_ */
