/*
 * semstream_b200.h -- C ABI of the B200-native semstream codec hot path.
 *
 * Drop-in boundary for the reference package `semstream`
 * (/root/reference/pkg/src/semstream, a pure numpy/scipy implementation).
 * Each entry point below replaces one reference function (cited file:line,
 * relative to pkg/src/semstream/) and reproduces its results bit-for-bit on
 * the same inputs.  A maintainer binds them from Python with ctypes; see
 * INTEGRATION.md.
 *
 * Conventions
 *   - All array pointers are DEVICE pointers owned by the caller (no
 *     allocation, no global state inside the library).  `stream` is a
 *     cudaStream_t passed as void*; every call is stream-ordered and
 *     non-blocking.  Calls are thread-safe for distinct (stream, buffers).
 *   - Return value: SST_OK (0) or a negative SST_ERR_* code for argument /
 *     launch errors.  Per-packet problems are reported in per-packet status
 *     words (SST_PKT_*), never as call failures.
 *   - Layouts (row-major, C order):
 *       frames      float32 [n][H][W][3]            (video.py:20-54 Frame)
 *       tokens      float64 [m][H'][W'][C]          (codec.py:49-91 TokenMatrix.values)
 *       token mask  uint8   [m][H'][W']  1 = valid  (TokenMatrix.mask)
 *       GoP batch   frames [G][9][H][W][3]; tokens [G][2][H'][W'][12] (I then P)
 *   - dtype of the arithmetic: float64 where the reference is float64,
 *     float32 storage where the reference stores float32.
 */
#ifndef SEMSTREAM_B200_H_
#define SEMSTREAM_B200_H_

#include <stdint.h>

#if defined(__GNUC__)
#define SST_API __attribute__((visibility("default")))
#else
#define SST_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* 3: + raw-rgb24 (sst_encode_u8, sst_upscale_blend_u8) and the decoder-fused
 * reconstruction (sst_unpack_tokens, sst_upscale_blend_tok, SstPrevTokDesc);
 * earlier entry points unchanged */
#define SST_ABI_VERSION 3

/* call status */
#define SST_OK 0
#define SST_ERR_ARG (-1)         /* bad shape / scale / pointer */
#define SST_ERR_ROWS_16BIT (-2)  /* > 65535 token rows: transport.py:245-246 "16-bit" */
#define SST_ERR_CUDA (-3)        /* CUDA runtime / launch failure */
#define SST_ERR_UNSUPPORTED (-4) /* e.g. channel count the kernel does not handle */

/* per-packet status (parse_packet, transport.py:154-218; reassemble, 274-305) */
#define SST_PKT_OK 0
#define SST_PKT_SHORT 1        /* "packet shorter than its checksum" */
#define SST_PKT_CRC 2          /* "crc32 mismatch" */
#define SST_PKT_BODY_SHORT 3   /* "packet body too short" */
#define SST_PKT_MAGIC 4        /* "bad magic" */
#define SST_PKT_VERSION 5      /* "unsupported version" */
#define SST_PKT_KIND 6         /* not a token packet (kind holds the raw kind byte) */
#define SST_PKT_HDR_TRUNC 7    /* "token packet header truncated" */
#define SST_PKT_MASK_TRUNC 8   /* "token packet mask truncated" */
#define SST_PKT_PAYLOAD_LEN 9  /* "payload length != popcount(mask)*C" */
#define SST_PKT_NEG_RANGE 10   /* "negative quantization range" */
#define SST_PKT_ABSENT 11      /* slot not present (lost in the network) */
#define SST_PKT_FOREIGN 12     /* kind / gop_id differ from the routed matrix (reassemble ValueError) */
#define SST_PKT_ROW_RANGE 13   /* row >= H': discarded, counted corrupt */
#define SST_PKT_DUP 14         /* duplicate row: a packet that arrived earlier wins */
#define SST_PKT_SHAPE 15       /* width / channel count incompatible with the matrix */

/* Parsed token-packet header (TokenPacket fields, transport.py:83-95). */
typedef struct SstPacketInfo {
  int32_t status;      /* SST_PKT_* */
  int32_t kind;        /* 0 = I, 1 = P */
  uint32_t gop_id;
  int32_t row;
  int32_t width;       /* width_tokens W' */
  int32_t channels;    /* C */
  int32_t scale;
  int32_t valid;       /* popcount(mask) */
  float qmin;          /* quant_min as carried on the wire */
  float qrange;        /* quant_range */
  int32_t mask_off;    /* byte offset of the mask inside the packet */
  int32_t payload_off; /* byte offset of the payload inside the packet */
  double dqmin;        /* quant_min / quant_range used by dequantisation: the */
  double dqrange;      /* wire float32 widened (parse), or a caller's float64 */
} SstPacketInfo;

/* Previous GoP of a stream, for boundary blending (codec.py:278-296). */
typedef struct SstPrevDesc {
  const float* p_img;  /* previous GoP's concealed P image, [h][w][3] at its working res; NULL = none */
  int32_t h, w, s;     /* its working size and scale */
  int32_t reserved;
} SstPrevDesc;

/* The previous GoP's token matrices for the decoder-fused reconstruction
 * (sst_upscale_blend_tok): its I and P tokens [2][Ht][Wt][12] float64, the
 * validity of its P tokens [Ht][Wt] (0 = concealed by the I block), and its
 * working geometry. */
typedef struct SstPrevTokDesc {
  const double* tok;       /* NULL = first GoP of its stream, no blend */
  const uint8_t* pvalid;
  int32_t h, w, s, Ht, Wt;
  int32_t reserved;
} SstPrevTokDesc;

SST_API int sst_abi_version(void);

/* Wire size of one token packet: transport.py:221-226 token_packet_wire_size. */
SST_API int64_t sst_packet_wire_size(int width_tokens, int channels, int valid_count);

/* ---- scaling ------------------------------------------------------------ */

/* downscale_frame (codec.py:202-214) for n frames: s x s box mean with edge
 * replication; out is [n][ceil(H/s)][ceil(W/s)][3] float32. */
SST_API int sst_downscale(const float* frames, int64_t n, int H, int W, int s, float* out, void* stream);

/* upscale_frame + crop (codec.py:238-245, 264-266): bilinear x s, clip to
 * [0,1], float32, crop to (crop_h, crop_w) (<= s*h, s*w). */
SST_API int sst_upscale(const float* img, int64_t n, int h, int w, int s, int crop_h, int crop_w,
                float* out, void* stream);

/* bilinear_upscale (codec.py:217-235): raw float64 result, no clip. */
SST_API int sst_bilinear_f64(const double* img, int64_t n, int h, int w, int s, double* out, void* stream);

/* np.clip(x, 0, 1).astype(float32): epilogue of upscale_frame for a
 * user-supplied upscaler (codec.py:243-245). */
SST_API int sst_clip_cast(const double* x, int64_t count, float* out, void* stream);

/* blend_boundary (codec.py:278-296) for G GoP pairs: out = curr with frames
 * 0..n-1 replaced by alpha*prev[9-n+i-1] + (1-alpha)*curr[i-1], alpha=(n-i)/n.
 * prev, curr, out: [G][9][H][W][3]; out may alias curr. */
SST_API int sst_blend(const float* prev, const float* curr, int G, int H, int W, int n, float* out,
              void* stream);

/* K5 for GoPs whose 9 frames are all distinct (learned-tokenizer decoder):
 * img [G][9][h][w][3] -> out [G][9][H][W][3] (bilinear x s, clip, crop),
 * frames 0..n-1 blended with the previous GoP's frames 9-n..8 upscaled from
 * prev[g].p_img = that GoP's [9][h'][w'][3] working frames (blend_n <= 4).
 * Samples must be >= 0 (the decoder clamps to [0, 1]; the clip's lower bound
 * is then a no-op and is not evaluated).  Any W; the windows of img are read
 * by TMA when img is 16-byte aligned and w*3*4 % 16 == 0, else by cp.async. */
SST_API int sst_upscale_blend9(const float* img, int G, int h, int w, int s, int H, int W,
                               const SstPrevDesc* prev, int blend_n, float* out, void* stream);

/* The same for uint8 working frames q whose sample value is float(q / 255)
 * (the int8 learned tokenizer's decoder output, SST_LT_EPI_PIXELS_U8);
 * prev[g].p_img points at the previous GoP's uint8 frames.  Output identical
 * to sst_upscale_blend9 on the equivalent float32 frames. */
SST_API int sst_upscale_blend9_u8(const uint8_t* img, int G, int h, int w, int s, int H, int W,
                                  const SstPrevDesc* prev, int blend_n, float* out, void* stream);

/* ---- tokenizer ---------------------------------------------------------- */

/* scale_gop(down) (codec.py:248-254) fused with encode_gop (codec.py:143-157)
 * and token_similarity(P, I) (selection.py:33-52).
 *   frames: [G][9][H][W][3] full resolution; s in {1 (frames already at
 *   working resolution: plain encode_gop), 2, 3}.
 *   tok: [G][2][H'][W'][12] float64 (I, P); sim: [G][H'][W'] float64 or NULL.
 * H' = ceil(ceil(H/s)/8), W' = ceil(ceil(W/s)/8). */
SST_API int sst_encode(const float* frames, int G, int H, int W, int s, double* tok, double* sim,
               void* stream);

/* sst_encode that also writes the working frames it box-filters (the
 * downscaled GoP scale_gop(gop, s, "down"), codec.py:202-214 / 248-254) to
 * work: [G][9][ceil(H/s)][ceil(W/s)][3] float32, or NULL (= sst_encode).
 * The residual layer's `working` GoP (session.py:173-189) without a second
 * read of the full-resolution frames. */
SST_API int sst_encode_work(const float* frames, int G, int H, int W, int s, double* tok,
               double* sim, float* work, void* stream);

/* sst_encode_work over raw-rgb24 frames: frames [G][9][H][W][3] uint8, each
 * byte q standing for the float32 sample float32(q) / 255 that
 * load_raw_video builds from it (video.py:130-135) -- the reference CLI's
 * encode input (cli.py:52-61,78-92).  Tokens, similarities and the optional
 * float32 working frames are those of sst_encode_work on the converted
 * frames, bit for bit. */
SST_API int sst_encode_u8(const uint8_t* frames, int G, int H, int W, int s, double* tok,
               double* sim, float* work, void* stream);

/* decode_gop (codec.py:160-186): IDCT of I and P tokens, crop to (h, w),
 * clip, conceal invalid P blocks with I blocks.
 *   i_tok, p_tok: [G][H'][W'][12] (any batch stride via tok_stride elements);
 *   p_mask: [G][H'][W'] or NULL (all valid); out: [G][2][h][w][3] float32
 *   (I image, concealed P image). */
SST_API int sst_decode(const double* i_tok, const double* p_tok, int64_t tok_stride, const uint8_t* p_mask,
               int G, int Ht, int Wt, int h, int w, float* out, void* stream);

/* ---- selection ---------------------------------------------------------- */

/* token_similarity (selection.py:33-52) for n token pairs with C channels. */
SST_API int sst_similarity(const double* p, const double* i, int64_t n, int C, double* sim, void* stream);

/* token_similarity for a GoP batch: tok [G][2][n][C] (I then P), sim [G][n]. */
SST_API int sst_similarity_gop(const double* tok, int G, int64_t n, int C, double* sim, void* stream);

/* top_k_drop_mask (selection.py:55-67): per map g, mark the k[g] largest
 * similarities (ties: lower row-major index first).  k is a DEVICE int32[G];
 * kth (DEVICE double[G] or NULL) receives the k-th largest value. */
SST_API int sst_topk_mask(const double* sim, int G, int64_t n, const int32_t* k, uint8_t* drop,
                          double* kth, void* stream);

/* apply_token_mask (codec.py:189-196) in place: mask &= ~drop, values of
 * invalid positions set to 0.0. */
SST_API int sst_apply_mask(double* values, uint8_t* mask, const uint8_t* drop, int64_t n, int C,
                   void* stream);

/* Fused intelligent drop for a freshly encoded GoP batch: top_k_drop_mask on
 * sim[g] then apply_token_mask on the P tokens of tok[g] ([G][2][H'][W'][12]
 * layout).  Every token of an encoder batch is valid (codec.py:155-157), so
 * the P half of mask [G][2][H'][W'] is ASSIGNED: P mask = not dropped (k = 0
 * restores an all-true P mask); the I half is not touched.  Dropped P values
 * are zeroed.  drop: [G][H'][W'] out or NULL. */
SST_API int sst_select_drop(const double* sim, double* tok, uint8_t* mask, int G, int Ht, int Wt,
                    const int32_t* k, uint8_t* drop, void* stream);

/* ---- wire format -------------------------------------------------------- */

/* packetize_tokens + TokenPacket.to_bytes (transport.py:236-271, 97-102):
 * one sealed packet per token row, written to arena[(m*Ht + row)*slot].
 *   values [m][H'][W'][C], mask [m][H'][W'] (NULL = all valid); kind/gop_id/
 *   scale per matrix (DEVICE arrays, length m); lengths: int32 [m*H'].
 *   slot >= sst_packet_wire_size(W', C, W') and a multiple of 16. */
SST_API int sst_packetize(const double* values, const uint8_t* mask, int m, int Ht, int Wt, int C,
                  const uint8_t* kind, const uint32_t* gop_id, const uint8_t* scale,
                  uint8_t* arena, int64_t slot, int32_t* lengths, void* stream);

/* TokenPacket.to_bytes for packets given field-wise (transport.py:97-102):
 *   info[n] supplies kind/gop/row/width/channels/scale/qmin/qrange/valid;
 *   mask bits (ceil(width/8) bytes, MSB first) at masks + mask_off[i];
 *   payload (valid*channels bytes) at payload + payload_off[i];
 *   output at out + out_off[i], sst_packet_wire_size(width, channels, valid) bytes. */
SST_API int sst_serialize(const SstPacketInfo* info, const uint8_t* masks, const int64_t* mask_off,
                  const uint8_t* payload, const int64_t* payload_off, int64_t n, uint8_t* out,
                  const int64_t* out_off, void* stream);

/* parse_packet (transport.py:154-218) for n packets at buf+off[i]
 * of len[i] bytes.  present (NULL = all) marks delivered packets. */
SST_API int sst_parse(const uint8_t* buf, const int64_t* off, const int32_t* len, const uint8_t* present,
              int64_t n, SstPacketInfo* info, void* stream);

/* reassemble (transport.py:274-305, dequantized 108-112) into m matrices.
 *   target[i] = matrix the caller routed packet i to (arrival order = i);
 *   exp_kind / exp_gop: expected kind and gop_id per matrix (DEVICE, len m);
 *   winner: uint32 [m][H'] workspace; values/mask: outputs [m][H'][W'][C],
 *   [m][H'][W']; stats: int32 [m][2] = {corrupt, rows_received}.
 *   Packet status is updated in place (FOREIGN, ROW_RANGE, DUP). */
SST_API int sst_reassemble(const uint8_t* buf, const int64_t* off, SstPacketInfo* info,
                   const int32_t* target, int64_t n, int m, int Ht, int Wt, int C,
                   const uint8_t* exp_kind, const uint32_t* exp_gop, uint32_t* winner,
                   double* values, uint8_t* mask, int32_t* stats, void* stream);

/* reassemble x2 + decode_gop fused: the mask-aware decoder reads each token
 * straight out of the winning packet (no token matrix in HBM).
 *   packets routed per GoP g as target[i] = 2*g + kind; exp_gop[G];
 *   ws: device workspace of sst_unpack_decode_workspace(G, H', W') bytes
 *   (16-byte aligned); out: [G][2][h][w][3] float32 (I image, concealed P). */
SST_API int64_t sst_unpack_decode_workspace(int G, int Ht, int Wt);
/* The receiver's reassemble x 2 + TokenPacket.dequantized (transport.py:
 * 108-112, 274-305) WITHOUT the IDCT: dequantised I / P token matrices
 * tok [G][2][Ht][Wt][12] float64 (missing rows / tokens 0) and the P
 * validity pvalid [G][Ht][Wt] -- the input of sst_upscale_blend_tok, which
 * runs decode_gop's IDCT + concealment inside the reconstruction.  Same
 * routing, first-wins and stats as sst_unpack_decode (same workspace). */
SST_API int sst_unpack_tokens(const uint8_t* buf, const int64_t* off, SstPacketInfo* info,
               const int32_t* target, int64_t n, int G, int Ht, int Wt, const uint32_t* exp_gop,
               uint32_t* winner, int32_t* stats, void* ws, double* tok, uint8_t* pvalid, void* stream);

SST_API int sst_unpack_decode(const uint8_t* buf, const int64_t* off, SstPacketInfo* info,
                              const int32_t* target, int64_t n, int G, int Ht, int Wt, int h, int w,
                              const uint32_t* exp_gop, uint32_t* winner, int32_t* stats, void* ws,
                              float* out, void* stream);

/* ---- reconstruction ----------------------------------------------------- */

/* scale_gop(up, crop) (codec.py:255-269) + blend_boundary (codec.py:278-296)
 * fused, materialising all 9 output frames of each GoP.
 *   img: [G][2][h][w][3] (I image, concealed P image) at scale s;
 *   prev: DEVICE SstPrevDesc[G] (p_img NULL = first GoP of its stream, no
 *   blend) or NULL; requires blend_n <= 4 when any prev is set (the blended
 *   tail frames are then unblended P reconstructions of the previous GoP);
 *   out: [G][9][H][W][3]. */
SST_API int sst_upscale_blend(const float* img, int G, int h, int w, int s, int H, int W,
                      const SstPrevDesc* prev, int blend_n, float* out, void* stream);

/* sst_upscale_blend with decode_gop fused in (codec.py:131-140,160-186 +
 * 217-296): reads the dequantised token matrices of sst_unpack_tokens and,
 * per output band, runs the 4-coefficient IDCT, clip and I-concealment of
 * exactly the working-image window it upscales (and of the previous GoP's P
 * window, from its tokens), so the working images never round-trip through
 * HBM.  Output bit-identical to sst_unpack_decode + sst_upscale_blend.
 *   tok [G][2][Ht][Wt][12], pvalid [G][Ht][Wt]; prev: DEVICE
 *   SstPrevTokDesc[G] or NULL (blend_n <= 4); out [G][9][H][W][3] float32,
 *   8-byte aligned, W*3 even (else SST_ERR_UNSUPPORTED). */
SST_API int sst_upscale_blend_tok(const double* tok, const uint8_t* pvalid, int G, int Ht, int Wt,
                      int h, int w, int s, int H, int W, const SstPrevTokDesc* prev, int blend_n,
                      float* out, void* stream);

/* sst_upscale_blend with raw-rgb24 output: every output sample v is written
 * as the byte write_raw_video stores for it (video.py:139-143,
 * np.rint(v * 255.0).astype(np.uint8) on the float32 frame), i.e. the
 * reference CLI's decode output (cli.py:181).  out: [G][9][H][W][3] uint8. */
SST_API int sst_upscale_blend_u8(const float* img, int G, int h, int w, int s, int H, int W,
                      const SstPrevDesc* prev, int blend_n, uint8_t* out, void* stream);

/* ---- residual enhancement layer and range coder (f2) ------- */

/* compute_residual + aggregate_residual + sparsify_quantize
 * (residual.py:62-105) for G GoPs at working resolution:
 *   work [G][9][h][w][3] source frames, img [G][2][h][w][3] reconstruction
 *   (I frame, shared P frame); avg [G][n] float64 (or NULL); dense [G][n] int16
 *   quantised residual where kept else 0; mags [G][n] |avg| where kept else
 *   -1 (or NULL; the fit_to_budget ranking key); count int32[G] kept entries.
 *   n = h*w*3. */
SST_API int sst_residual(const float* work, const float* img, int G, int h, int w, double theta,
                         double step, double* avg, int16_t* dense, double* mags, int32_t* count,
                         void* stream);

/* aggregate_residual (residual.py:76-83): out[e] = (sum_t res[t][e]) / T,
 * summed sequentially from 0.0 in float64. */
SST_API int sst_mean_axis0(const double* res, int T, int64_t n, double* out, void* stream);

/* sparsify_quantize (residual.py:86-105) of given float64 averages [G][n]. */
SST_API int sst_sparsify(const double* avg, int G, int64_t n, double theta, double step,
                         int16_t* dense, double* mags, int32_t* count, void* stream);

/* apply_residual (residual.py:108-127): img[g][0..1] = clip(img + dense*step)
 * unless count[g] == 0 (reconstruction left untouched). */
SST_API int sst_apply_residual(float* img, const int16_t* dense, const int32_t* count, int G,
                               int h, int w, double step, void* stream);

/* compute_residual (residual.py:62-73): out[e] = (double)x[e] - (double)xh[e]. */
SST_API int sst_residual_diff(const float* x, const float* xh, int64_t n, double* out, void* stream);

/* SparseResidual.dense (residual.py:56-59): out[e] = (double)q[e] * step. */
SST_API int sst_dequant_i16(const int16_t* q, int64_t n, double step, double* out, void* stream);

/* out[e] = keep[e] ? dense[e] : 0 (fit_to_budget candidate scan). */
SST_API int sst_mask_scan(const int16_t* dense, const uint8_t* keep, int64_t total, int16_t* out,
                          void* stream);

/* rangecoder.encode_scan (rangecoder.py:75-94,155-185,238-239) for G scans of
 * n int16 samples: bytes to out + g*cap, length to out_len[g] (negative =
 * -(needed bytes) when cap is too small).  idx_ws: int64 [G][n] workspace. */
SST_API int sst_rc_encode(const int16_t* scans, int G, int64_t n, int64_t* idx_ws, uint8_t* out,
                          int64_t cap, int64_t* out_len, void* stream);

/* rangecoder.decode_scan (rangecoder.py:97-116,188-243): status[g] 0 ok,
 * 1 truncated, 2 zero run overruns, 3 value overruns, 4 symbol budget. */
SST_API int sst_rc_decode(const uint8_t* data, const int64_t* off, const int64_t* len, int G,
                          int64_t n, int16_t* scans, int32_t* status, void* stream);

/* rangecoder.encode_stream for explicit symbol lists (rangecoder.py:155-185):
 * stream g = syms[off[g] .. off[g]+len[g]); bytes to out + g*cap. */
SST_API int sst_rc_encode_symbols(const int32_t* syms, const int64_t* off, const int64_t* len,
                                  int G, uint8_t* out, int64_t cap, int64_t* out_len,
                                  void* stream);

/* rangecoder.decode_stream (rangecoder.py:188-235): symbols to syms (<= cap),
 * count to *nsym; status 0 ok, 1 truncated, 4 symbol budget, 7 capacity. */
SST_API int sst_rc_decode_symbols(const uint8_t* data, int64_t nbytes, int64_t max_symbols,
                                  int64_t cap, int32_t* syms, int64_t* nsym, int32_t* status,
                                  void* stream);

/* ---- learned tokenizer plug-in ----------------------
 * A causal spatio-temporal conv tokenizer with finite-scalar quantisation
 * (FSQ), plugged in at the reference's tokenizer hook
 * SessionConfig.tokenizer_encode / tokenizer_decode (session.py:57-61,
 * contract SPEC.md:165).  The reference ships no learned model,
 * so these entry points have no reference function to match: parity is
 * against the torch fp32 restatement in oracle/learned_oracle.py (unpinned).
 * Activations are bf16 channels-last [G][T][H'][W'][C]; the convolutions run
 * as tcgen05 implicit GEMMs (bf16 x bf16 -> fp32 in TMEM), operands by TMA. */

#define SST_LT_EPI_STORE 0   /* bf16 activation tensor (+bias, SiLU, +residual) */
#define SST_LT_EPI_FSQ 1     /* FSQ head: codes f64 [G][2][H'][W'][12], idx i32 [..][2], mask u8 */
#define SST_LT_EPI_PIXELS 2  /* unpatchify: frames f32 [G][9][h][w][3], clamp [0,1] */
#define SST_LT_EPI_PIXELS_U8 3 /* (sst_lt8_conv) unpatchify to uint8 q: sample = float(q / 255) */

typedef struct SstConvDesc {
  const void* in;          /* bf16 [G][in_T][in_H][in_W][in_C], in_C % 64 == 0 */
  int32_t in_C, in_W, in_H, in_T;
  int32_t G, Ht, Wt;       /* output token grid per latent frame */
  int32_t t_lo, t_cnt;     /* output latent frames t_lo .. t_lo+t_cnt-1 */
  int32_t n_taps;          /* <= 27 */
  int32_t taps[27][3];     /* (dt, dy, dx) input offsets per tap; K order = tap-major, channel-minor */
  const void* weight;      /* bf16 [N][K], K = n_taps * in_C */
  int32_t N, K;
  const float* bias;       /* fp32 [N], 16-byte aligned */
  int32_t epi, act;        /* SST_LT_EPI_*; act 1 = SiLU (STORE only) */
  const void* residual;    /* STORE: bf16, same layout as out, or NULL */
  void* out;               /* STORE: bf16 [G][out_T][Ht][Wt][N] */
  int32_t out_T;
  double* codes;           /* FSQ */
  int32_t* idx;
  uint8_t* mask;
  float* frames;           /* PIXELS: frame f = frame_base + N-tile index (192 columns per frame) */
  int32_t h, w, frame_base;
  /* int8 layers (sst_lt8_conv only; ignored by sst_lt_conv): in / weight /
   * residual / out are int8, in_C % 128 == 0, accumulators int32 (exact) */
  int32_t shift;           /* requantisation: y = clamp((acc + b + 2^(shift-1)) >> shift, -127, 127) */
  const int32_t* bias_i32; /* int32 [N], 16-byte aligned */
  const int8_t* act_lut;   /* act 1: y = act_lut[y + 128] (the SiLU table) */
} SstConvDesc;

/* One convolution layer (implicit GEMM on tcgen05). */
SST_API int sst_lt_conv(const SstConvDesc* d, void* stream);

/* Box downscale (codec.py:202-214, bit-exact) + edge pad to 8 (codec.py:99-105)
 * + 8x8 patchify to bf16: pI [G][H'][W'][192] (frame 0), pP [G][H'][W'][1536]
 * (frames 1..8), K order (frame, py, px, colour).  s in {1, 2, 3}. */
SST_API int sst_lt_patchify(const float* frames, int G, int H, int W, int s, void* pI, void* pP,
                            void* stream);

/* Mask-aware decoder input: snap the received codes (tokens f64
 * [G][2][H'][W'][12], e.g. reassemble output) to the FSQ grid, conceal masked
 * P tokens with the co-located I token (codec.py:176-180 semantics in latent
 * space) and write bf16 [G][2][H'][W'][64] (channels 12..63 zero). */
SST_API int sst_lt_dec_in(const double* tok, const uint8_t* mask, int G, int Ht, int Wt, void* out,
                          void* stream);

/* reassemble x2 fused with the learned decoder's input stage: packets routed
 * as for sst_unpack_decode (ws = sst_unpack_decode_workspace bytes); writes
 * the snapped, concealed bf16 [G][2][H'][W'][64] decoder input directly. */
SST_API int sst_lt_unpack_dec_in(const uint8_t* buf, const int64_t* off, SstPacketInfo* info,
                                 const int32_t* target, int64_t n, int G, int Ht, int Wt,
                                 const uint32_t* exp_gop, uint32_t* winner, int32_t* stats,
                                 void* ws, void* out, void* stream);

/* Causal spatio-temporal window attention core of the learned tokenizer:
 * qkv bf16 [G][2][H'][W'][3D] (Q | K | V, head-major 64-dim heads, from one
 * 1x1 sst_lt_conv), out bf16 [G][2][H'][W'][D].  Each query attends to the
 * valid tokens of its 8x8 window in latent frames <= its own (softmax in
 * fp32, scale 1/8). */
SST_API int sst_lt_attn(const void* qkv, int G, int Ht, int Wt, int D, void* out, void* stream);

/* qkv projection fused with the attention core: h bf16 [G][2][H'][W'][D]
 * (the block input), w_qkv bf16 [3D][D], b_qkv fp32 [3D] (16-byte aligned) -> out bf16
 * [G][2][H'][W'][D]; same result definition as a 1x1 sst_lt_conv (bf16 qkv)
 * followed by sst_lt_attn. */
SST_API int sst_lt_attn_fused(const void* h, const void* w_qkv, const float* b_qkv, int G, int Ht,
                              int Wt, int D, void* out, void* stream);

/* ---- int8 learned tokenizer (exact integer arithmetic, kind::i8) ---------
 * The same plug-in network shape with int8 activations / weights and int32
 * tensor-core accumulation: bit-identical to oracle/learned_i8_oracle.py
 * (which documents the arithmetic).  Activations int8 channels-last
 * [G][T][H'][W'][C], C % 128 == 0. */

/* One int8 layer: SstConvDesc with the int8 fields (shift, bias_i32,
 * act_lut); epi STORE (requantise, SiLU table, saturating residual add, int8
 * out), FSQ (N = 16: q = clamp((acc + b) >> shift, -L/2, L-1-L/2), codes
 * q/(L/2) f64, mixed-radix indices, mask = 1) or PIXELS (clamp(round-shift,
 * 0, 255) / 255 float32 frames). */
SST_API int sst_lt8_conv(const SstConvDesc* d, void* stream);

/* Box downscale (bit-exact) + edge pad + 8x8 patchify to int8
 * rint(px * 255) - 128: pI [G][H'][W'][256] (192 used, rest zero), pP
 * [G][H'][W'][1536]. */
SST_API int sst_lt8_patchify(const float* frames, int G, int H, int W, int s, void* pI, void* pP,
                             void* stream);

/* The same through the integer 3-D Haar wavelet front end (Cosmos' first
 * stage): per 8x8 patch, three temporal levels over the eight
 * P frames, then three spatial levels (horizontal, then vertical) on every
 * frame slot; pairs (a, b) -> ((a + b) >> 1, (a - b) >> 1), Mallat layout,
 * int8 throughout.  Same output layout; pP must be 16-byte aligned too. */
SST_API int sst_lt8_patchify_haar(const float* frames, int G, int H, int W, int s, void* pI,
                                  void* pP, void* stream);

/* Causal 8x8-window attention core, 128-dim heads, integer softmax:
 * qkv int8 [G][2][H'][W'][3D] -> out int8 [G][2][H'][W'][D]; shift and
 * exp_lut (uint8[256]) as in the oracle. */
SST_API int sst_lt8_attn(const void* qkv, int G, int Ht, int Wt, int D, int shift,
                         const uint8_t* exp_lut, void* out, void* stream);

/* The same with GLOBAL causal attention: every query attends all valid tokens
 * of the latent frames <= its own (full H' x W' frames, no windows); keys
 * stream through shared memory in 128-token tiles (two passes: row max, then
 * P / sum / O += P V on tcgen05), bit-exact to the oracle. */
SST_API int sst_lt8_attn_global(const void* qkv, int G, int Ht, int Wt, int D, int shift,
                                const uint8_t* exp_lut, void* out, void* stream);

/* Decoder input from a token matrix (plug-in path): received f64 codes
 * [G][2][H'][W'][12] + mask -> snapped, concealed codes (ws: G*2*H'*W'*16
 * bytes) -> the first layer's gathered (2,3,3) neighbourhood, int8
 * [G][2][H'][W'][256]. */
SST_API int sst_lt8_dec_in(const double* tok, const uint8_t* mask, int G, int Ht, int Wt, void* ws,
                           void* out, void* stream);

/* The same straight from the winning row packets (reassemble x2 fused with
 * the decoder input; packets routed as for sst_unpack_decode). */
SST_API int64_t sst_lt8_unpack_workspace(int G, int Ht, int Wt);
SST_API int sst_lt8_unpack_dec_in(const uint8_t* buf, const int64_t* off, SstPacketInfo* info,
                                  const int32_t* target, int64_t n, int G, int Ht, int Wt,
                                  const uint32_t* exp_gop, uint32_t* winner, int32_t* stats,
                                  void* ws, void* out, void* stream);

/* ---- metrics ------------------------------------------------------------ */

/* np.mean over `elems` float64 per-pixel differences of n frame pairs
 * a[i], b[i] (float32 [n][elems]): mode 0 = (a-b)^2 (mse, video.py:265-270;
 * gop_psnr's per-frame errors, video.py:318-322; the l2 flicker norm),
 * mode 1 = |a-b| (boundary_flicker l1, video.py:285-304;
 * inter_frame_consistency, video.py:307-315).  Summed in numpy's pairwise
 * order from 0.0, divided by elems: bit-identical to the reference. */
SST_API int sst_mean_diff(const float* a, const float* b, int64_t n, int64_t elems, int mode,
                          double* out, void* stream);

/* mse (video.py:265-270) per frame pair = sst_mean_diff mode 0. */
SST_API int sst_mse(const float* a, const float* b, int64_t n, int64_t elems, double* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SEMSTREAM_B200_H_ */
