// K4: mask-aware decoder (decode_gop, codec.py:160-186; _detokenize,
// codec.py:131-140), optionally fused with reassemble (transport.py:274-305).
//
// One CTA decodes 8 consecutive tokens of one token row for both layers:
//   tokens (from a token matrix, or dequantised straight out of the winning
//   row packet -- the "first conv" of the mask-aware decoder consumes the
//   packet scatter directly, no token matrix is materialised)
//   -> 4-coefficient IDCT along y (ducc0 order, fct 1/16) into smem
//   -> IDCT along x per pixel row, clip to [0,1]
//   -> temporal-reference concealment (invalid P block <- I block)
//   -> float32 working-resolution I and P images, cropped to (h, w).
#include <cuda_bf16.h>

#include "common.cuh"
#include "dct8.cuh"

namespace sst {

// Winning packet of one matrix row, resolved once by k_rowprep
struct RowInfo {
  int64_t payload;   // byte offset of the payload in the packet buffer
  double qmin;       // quant_min
  double step;       // quant_range / 255.0 (transport.py:112)
  int32_t ok;
  int32_t pad;
};

// One warp per matrix row: validate the winner's shape, count the row as
// received, and turn its MSB-first mask into per-token payload slots.
__global__ void __launch_bounds__(256)
    k_rowprep(const int64_t* __restrict__ off, SstPacketInfo* info, const uint8_t* __restrict__ buf,
              const uint32_t* __restrict__ winner, int64_t nrows, int Ht, int Wt,
              RowInfo* __restrict__ rows, int32_t* __restrict__ tokoff, int32_t* stats) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= nrows) return;
  const uint32_t win = winner[r];
  bool ok = win != 0xFFFFFFFFu;
  RowInfo ri{0, 0.0, 0.0, 0, 0};
  const uint8_t* mb = nullptr;
  if (ok) {
    SstPacketInfo& p = info[win];
    const uint8_t* pkt = buf + off[win];
    mb = pkt + p.mask_off;
    // shape contract of the fused path: W' tokens of 12 channels
    bool bad = p.channels != kChannels || p.width < Wt;
    for (int x = Wt + lane; !bad && x < p.width; x += 32)
      if ((mb[x >> 3] >> (7 - (x & 7))) & 1) bad = true;
    bad = __any_sync(0xffffffffu, bad);
    if (bad) {
      if (lane == 0) p.status = SST_PKT_SHAPE;
      ok = false;
    } else {
      ri.payload = off[win] + p.payload_off;
      ri.qmin = p.dqmin;
      ri.step = p.dqrange / 255.0;
      ri.ok = 1;
      if (lane == 0) atomicAdd(&stats[2 * (r / Ht) + 1], 1);   // rows_received
    }
  }
  if (lane == 0) rows[r] = ri;
  int running = 0;
  for (int base = 0; base < Wt; base += 32) {
    const int x = base + lane;
    const bool v = ok && x < Wt && ((mb[x >> 3] >> (7 - (x & 7))) & 1);
    const unsigned bal = __ballot_sync(0xffffffffu, v);
    if (x < Wt) tokoff[r * Wt + x] = v ? running + __popc(bal & ((1u << lane) - 1u)) : -1;
    running += __popc(bal);
  }
}

constexpr int kDecTok = 16;     // tokens per CTA
constexpr int kDecThreads = 384; // = kDecTok * 3 channels * 8 pixel rows

struct DecArgs {
  // token-matrix source
  const double* i_tok;
  const double* p_tok;
  int64_t tok_stride;          // elements between consecutive GoPs in i_tok / p_tok
  const uint8_t* p_mask;       // [G][Ht][Wt] or null
  // packet source (when buf != null)
  const uint8_t* buf;
  const int64_t* off;
  SstPacketInfo* info;
  const uint32_t* winner;      // [G*2][Ht]
  int32_t* stats;              // [G*2][2]
  const struct RowInfo* rows;  // [G*2][Ht] winning packet per matrix row
  const int32_t* tokoff;       // [G*2][Ht][Wt] payload slot of each token or -1
  int G, Ht, Wt, h, w;
  float* out;                  // [G][2][h][w][3]
};

template <bool kFromPackets>
__global__ void __launch_bounds__(kDecThreads) k_decode(DecArgs a) {
  __shared__ double tok[2][kDecTok][kChannels];
  __shared__ uint8_t valid[kDecTok];
  // column-IDCT results for block columns 0, 1: [img][y][x][tok*3 + ch]
  // (token/channel innermost so a warp's reads are consecutive: no conflicts)
  __shared__ double s1[2][8][2][kDecTok * 3];
  __shared__ double zc[8];                         // column IDCT of an all-zero column
  __shared__ float pix[2][8][kDecTok * 8][3];      // output tile

  const int tid = threadIdx.x;
  const int tx0 = blockIdx.x * kDecTok;
  const int ty = blockIdx.y;
  const int g = blockIdx.z;

  // ---- 1. gather the tokens ----
  if (kFromPackets) {
    // every thread dequantises one (layer, token, channel) straight from the
    // winning packet's payload (transport.py:108-112, 296-302)
    for (int e = tid; e < 2 * kDecTok * kChannels; e += kDecThreads) {
      const int im = e / (kDecTok * kChannels);
      const int t = (e / kChannels) % kDecTok;
      const int c = e % kChannels;
      const int tx = tx0 + t;
      const int64_t r = ((int64_t)g * 2 + im) * a.Ht + ty;
      const int slot = tx < a.Wt ? a.tokoff[r * a.Wt + tx] : -1;
      double v = 0.0;
      if (slot >= 0) {
        const RowInfo& ri = a.rows[r];
        v = ri.qmin + (double)a.buf[ri.payload + (int64_t)slot * kChannels + c] * ri.step;
      }
      tok[im][t][c] = v;
      if (im == 1 && c == 0) valid[t] = slot >= 0 ? 1 : 0;
    }
  } else {
    for (int e = tid; e < 2 * kDecTok * kChannels; e += kDecThreads) {
      int im = e / (kDecTok * kChannels);
      int t = (e / kChannels) % kDecTok;
      int c = e % kChannels;
      int tx = tx0 + t;
      double v = 0.0;
      if (tx < a.Wt) {
        const double* src = (im == 0 ? a.i_tok : a.p_tok) + (int64_t)g * a.tok_stride;
        v = src[((int64_t)ty * a.Wt + tx) * kChannels + c];
      }
      tok[im][t][c] = v;
    }
    if (tid < kDecTok) {
      int tx = tx0 + tid;
      valid[tid] = (tx < a.Wt && a.p_mask) ? a.p_mask[((int64_t)g * a.Ht + ty) * a.Wt + tx] : 1;
    }
  }
  __syncthreads();

  // ---- 2. IDCT along y for every block column x (coefficients at (0,0),
  //         (0,1), (1,0), (2,0); codec.py:134-138).  Columns 2..7 hold only
  //         zeros, so their (identical) result is computed once. ----
  for (int it = tid; it < 2 * kDecTok * 3 * 2 + 1; it += kDecThreads) {
    double c[8];
#pragma unroll
    for (int y = 0; y < 8; ++y) c[y] = 0.0;
    if (it == 2 * kDecTok * 3 * 2) {
      dct3_8<true>(c, 1.0 / 16.0);
#pragma unroll
      for (int y = 0; y < 8; ++y) zc[y] = c[y];
      continue;
    }
    int im = it / (kDecTok * 6);
    int t = (it / 6) % kDecTok;
    int ch = (it / 2) % 3;
    int x = it % 2;
    const double* v = tok[im][t] + ch * 4;
    if (x == 0) { c[0] = v[0]; c[1] = v[2]; c[2] = v[3]; }
    else { c[0] = v[1]; }
    dct3_8<true>(c, 1.0 / 16.0);
#pragma unroll
    for (int y = 0; y < 8; ++y) s1[im][y][x][t * 3 + ch] = c[y];
  }
  __syncthreads();

  // ---- 3. IDCT along x per pixel row, clip, conceal ----
  for (int it = tid; it < kDecTok * 3 * 8; it += kDecThreads) {
    const int y = it / (kDecTok * 3);
    const int tc = it % (kDecTok * 3);
    const int t = tc / 3, ch = tc % 3;
    double ci[8], cp[8];
    ci[0] = s1[0][y][0][tc]; ci[1] = s1[0][y][1][tc];
    cp[0] = s1[1][y][0][tc]; cp[1] = s1[1][y][1][tc];
    const double z = zc[y];
#pragma unroll
    for (int x = 2; x < 8; ++x) { ci[x] = z; cp[x] = z; }
    dct3_8<false>(ci, 1.0);
    dct3_8<false>(cp, 1.0);
    const bool keep_p = valid[t] != 0;
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      double iv = clip01(ci[x]);
      double pv = keep_p ? clip01(cp[x]) : iv;
      pix[0][y][t * 8 + x][ch] = (float)iv;
      pix[1][y][t * 8 + x][ch] = (float)pv;
    }
  }
  __syncthreads();

  // ---- 4. store the cropped tile (16-byte stores when rows are aligned) ----
  const int y0 = ty * 8, x0 = tx0 * 8;
  const int rows = min(8, a.h - y0);
  const int nq = min(kDecTok * 8, a.w - x0) * 3;          // floats per tile row
  constexpr int kRowF = kDecTok * 8 * 3;
  if ((a.w & 3) == 0) {
    constexpr int kRow4 = kRowF / 4;
    for (int e = tid; e < 2 * 8 * kRow4; e += kDecThreads) {
      const int im = e / (8 * kRow4);
      const int r = (e / kRow4) % 8;
      const int q = (e % kRow4) * 4;
      if (r >= rows || q >= nq) continue;
      const float* srcp = &pix[im][r][0][0] + q;
      float* dstp = a.out + ((((int64_t)g * 2 + im) * a.h + y0 + r) * a.w + x0) * 3 + q;
      if (q + 4 <= nq) {
        *reinterpret_cast<float4*>(dstp) = make_float4(srcp[0], srcp[1], srcp[2], srcp[3]);
      } else {
        for (int u = 0; u < nq - q; ++u) dstp[u] = srcp[u];
      }
    }
  } else {
    for (int e = tid; e < 2 * 8 * kRowF; e += kDecThreads) {
      const int im = e / (8 * kRowF);
      const int r = (e / kRowF) % 8;
      const int q = e % kRowF;
      if (r < rows && q < nq)
        a.out[((((int64_t)g * 2 + im) * a.h + y0 + r) * a.w + x0) * 3 + q] = (&pix[im][r][0][0])[q];
    }
  }
}

// ---- packets -> dequantised token matrices (for K5 with the decoder fused) ----
// reassemble x 2 + TokenPacket.dequantized (transport.py:108-112,274-305):
// the I and P token matrices [G][2][Ht][Wt][12] float64 (missing rows and
// tokens 0) and the P validity [G][Ht][Wt] -- what K4b's gather stage holds
// in shared memory, written out so that the IDCT can run inside K5
// (sst_upscale_blend_tok) right where the working image is consumed.
__global__ void k_unpack_tok(const uint8_t* __restrict__ buf, const RowInfo* __restrict__ rows,
                             const int32_t* __restrict__ tokoff, int Ht, int Wt, double* __restrict__ tok,
                             uint8_t* __restrict__ pvalid) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= Wt * kChannels) return;
  const int tx = e / kChannels, c = e - tx * kChannels;
  const int ty = blockIdx.y, m = blockIdx.z;                  // m = 2 g + im
  const int64_t r = (int64_t)m * Ht + ty;
  const int slot = tokoff[r * Wt + tx];
  double v = 0.0;
  if (slot >= 0) {
    const RowInfo& ri = rows[r];
    v = ri.qmin + (double)buf[ri.payload + (int64_t)slot * kChannels + c] * ri.step;
  }
  tok[(r * Wt + tx) * kChannels + c] = v;
  if ((m & 1) && c == 0) pvalid[((int64_t)(m >> 1) * Ht + ty) * Wt + tx] = slot >= 0 ? 1 : 0;
}

int route_packets(SstPacketInfo* info, const int32_t* target, int64_t n, int m, int Ht,
                  const uint8_t* exp_kind, const uint32_t* exp_gop, uint32_t* winner,
                  int32_t* stats, cudaStream_t st);

}  // namespace sst

using namespace sst;

extern "C" int sst_decode(const double* i_tok, const double* p_tok, int64_t tok_stride,
                          const uint8_t* p_mask, int G, int Ht, int Wt, int h, int w, float* out,
                          void* stream) {
  if (G < 0 || Ht <= 0 || Wt <= 0 || h <= 0 || w <= 0) return SST_ERR_ARG;
  if (h > Ht * 8 || w > Wt * 8) return SST_ERR_ARG;
  if (G == 0) return SST_OK;
  if (!i_tok || !p_tok || !out) return SST_ERR_ARG;
  if (Ht > 65535 || G > 65535) return SST_ERR_ARG;
  DecArgs a{};
  a.i_tok = i_tok; a.p_tok = p_tok; a.tok_stride = tok_stride; a.p_mask = p_mask;
  a.G = G; a.Ht = Ht; a.Wt = Wt; a.h = h; a.w = w; a.out = out;
  dim3 grid(ceil_div(Wt, kDecTok), Ht, G);
  k_decode<false><<<grid, kDecThreads, 0, static_cast<cudaStream_t>(stream)>>>(a);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int64_t sst_unpack_decode_workspace(int G, int Ht, int Wt) {
  const int64_t rows = 2 * (int64_t)G * Ht;
  return rows * (int64_t)sizeof(RowInfo) + rows * Wt * 4;
}

extern "C" int sst_unpack_tokens(const uint8_t* buf, const int64_t* off, SstPacketInfo* info,
                                 const int32_t* target, int64_t n, int G, int Ht, int Wt,
                                 const uint32_t* exp_gop, uint32_t* winner, int32_t* stats, void* ws,
                                 double* tok, uint8_t* pvalid, void* stream) {
  if (n < 0 || G < 0 || Ht <= 0 || Wt <= 0) return SST_ERR_ARG;
  if (G == 0) return SST_OK;
  if (!exp_gop || !winner || !stats || !tok || !pvalid || !ws) return SST_ERR_ARG;
  if (n > 0 && (!buf || !off || !info || !target)) return SST_ERR_ARG;
  if (Ht > 65535 || G > 32767) return SST_ERR_ARG;
  if (reinterpret_cast<uintptr_t>(ws) & 15) return SST_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = route_packets(info, target, n, 2 * G, Ht, nullptr, exp_gop, winner, stats, st);
  if (rc != SST_OK) return rc;
  const int64_t nrows = 2 * (int64_t)G * Ht;
  RowInfo* rows = static_cast<RowInfo*>(ws);
  int32_t* tokoff = reinterpret_cast<int32_t*>(rows + nrows);
  k_rowprep<<<(unsigned)ceil_div64(nrows, 8), 256, 0, st>>>(off, info, buf, winner, nrows, Ht, Wt,
                                                            rows, tokoff, stats);
  SST_LAUNCH_CHECK();
  dim3 grid(ceil_div(Wt * kChannels, 256), Ht, 2 * G);
  k_unpack_tok<<<grid, 256, 0, st>>>(buf, rows, tokoff, Ht, Wt, tok, pvalid);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_unpack_decode(const uint8_t* buf, const int64_t* off, SstPacketInfo* info,
                                 const int32_t* target, int64_t n, int G, int Ht, int Wt, int h,
                                 int w, const uint32_t* exp_gop, uint32_t* winner, int32_t* stats,
                                 void* ws, float* out, void* stream) {
  if (n < 0 || G < 0 || Ht <= 0 || Wt <= 0 || h <= 0 || w <= 0) return SST_ERR_ARG;
  if (h > Ht * 8 || w > Wt * 8) return SST_ERR_ARG;
  if (G == 0) return SST_OK;
  if (!exp_gop || !winner || !stats || !out || !ws) return SST_ERR_ARG;
  if (n > 0 && (!buf || !off || !info || !target)) return SST_ERR_ARG;
  if (Ht > 65535 || G > 65535) return SST_ERR_ARG;
  if (reinterpret_cast<uintptr_t>(ws) & 15) return SST_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = route_packets(info, target, n, 2 * G, Ht, nullptr, exp_gop, winner, stats, st);
  if (rc != SST_OK) return rc;
  const int64_t nrows = 2 * (int64_t)G * Ht;
  RowInfo* rows = static_cast<RowInfo*>(ws);
  int32_t* tokoff = reinterpret_cast<int32_t*>(rows + nrows);
  k_rowprep<<<(unsigned)ceil_div64(nrows, 8), 256, 0, st>>>(off, info, buf, winner, nrows, Ht, Wt,
                                                            rows, tokoff, stats);
  SST_LAUNCH_CHECK();
  DecArgs a{};
  a.buf = buf; a.off = off; a.info = info; a.winner = winner; a.stats = stats;
  a.rows = rows; a.tokoff = tokoff;
  a.G = G; a.Ht = Ht; a.Wt = Wt; a.h = h; a.w = w; a.out = out;
  dim3 grid(ceil_div(Wt, kDecTok), Ht, G);
  k_decode<true><<<grid, kDecThreads, 0, st>>>(a);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

// ---- learned tokenizer: packets -> decoder input ----------------
// The mask-aware learned decoder's input stage fused with reassembly: one
// thread per latent token dequantises its 12 FSQ-code channels straight out of
// the winning row packet (transport.py:108-112: qmin + raw * (qrange / 255)),
// conceals a missing P token with the co-located I token, snaps the values
// back onto the FSQ grid and writes the bf16 [G][2][H'][W'][64] input of the
// first decoder convolution -- no token matrix is materialised.
namespace sst {
__device__ __forceinline__ int lt_levels(int i) { return (i % 6) < 3 ? 8 : 5; }

__global__ void k_lt_unpack_dec_in(const uint8_t* __restrict__ buf, const RowInfo* __restrict__ rows,
                                   const int32_t* __restrict__ tokoff, int G, int Ht, int Wt,
                                   __nv_bfloat16* __restrict__ out) {
  const int64_t n = (int64_t)Ht * Wt;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)G * 2 * n) return;
  const int64_t pos = idx % n;
  const int64_t gt = idx / n;
  const int t = (int)(gt % 2);
  const int64_t g = gt / 2;
  const int y = (int)(pos / Wt), x = (int)(pos % Wt);
  int64_t r = (g * 2 + t) * Ht + y;
  int slot = tokoff[r * Wt + x];
  if (t == 1 && slot < 0) {               // conceal with the co-located I token
    r = (g * 2) * Ht + y;
    slot = tokoff[r * Wt + x];
  }
  uint4 o[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) o[q] = make_uint4(0, 0, 0, 0);
  if (slot >= 0) {
    const RowInfo ri = rows[r];
    const uint8_t* p = buf + ri.payload + (int64_t)slot * kChannels;
    __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(o);
#pragma unroll
    for (int i = 0; i < kChannels; ++i) {
      const double v = ri.qmin + (double)p[i] * ri.step;
      const int L = lt_levels(i), hw = L / 2;
      double q = rint(v * (double)hw);
      q = fmin(fmax(q, (double)-hw), (double)(L - 1 - hw));
      ob[i] = __float2bfloat16_rn((float)(q / (double)hw));
    }
  }
  uint4* op = reinterpret_cast<uint4*>(out + idx * 64);
#pragma unroll
  for (int q = 0; q < 8; ++q) op[q] = o[q];
}
}  // namespace sst

extern "C" int sst_lt_unpack_dec_in(const uint8_t* buf, const int64_t* off, SstPacketInfo* info,
                                    const int32_t* target, int64_t n, int G, int Ht, int Wt,
                                    const uint32_t* exp_gop, uint32_t* winner, int32_t* stats,
                                    void* ws, void* out, void* stream) {
  if (n < 0 || G < 0 || Ht <= 0 || Wt <= 0) return SST_ERR_ARG;
  if (G == 0) return SST_OK;
  if (!exp_gop || !winner || !stats || !out || !ws) return SST_ERR_ARG;
  if (n > 0 && (!buf || !off || !info || !target)) return SST_ERR_ARG;
  if (Ht > 65535 || G > 65535) return SST_ERR_ARG;
  if (reinterpret_cast<uintptr_t>(ws) & 15) return SST_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = route_packets(info, target, n, 2 * G, Ht, nullptr, exp_gop, winner, stats, st);
  if (rc != SST_OK) return rc;
  const int64_t nrows = 2 * (int64_t)G * Ht;
  RowInfo* rows = static_cast<RowInfo*>(ws);
  int32_t* tokoff = reinterpret_cast<int32_t*>(rows + nrows);
  k_rowprep<<<(unsigned)ceil_div64(nrows, 8), 256, 0, st>>>(off, info, buf, winner, nrows, Ht, Wt,
                                                            rows, tokoff, stats);
  SST_LAUNCH_CHECK();
  const int64_t total = nrows * Wt;
  k_lt_unpack_dec_in<<<(unsigned)ceil_div64(total, 256), 256, 0, st>>>(
      buf, rows, tokoff, G, Ht, Wt, static_cast<__nv_bfloat16*>(out));
  SST_LAUNCH_CHECK();
  return SST_OK;
}

// ---- int8 learned tokenizer: decoder input (learned_i8.py) -------
// Received codes -> snapped, concealed FSQ levels q (x16, int8) per token
// ([G][2][H'][W'][16], channels 12..15 zero), then the first decoder layer's
// (2,3,3) neighbourhood gathered tap-major into 2 x 9 x 12 = 216 (+40 zero)
// channels, so that layer is one K = 256 int8 GEMM
// (oracle/learned_i8_oracle.py snap_codes / dec_input).
namespace sst {

__device__ __forceinline__ int8_t l8_snap(double v, int i) {
  const int L = lt_levels(i), hw = L / 2;
  double q = rint(v * (double)hw);
  q = fmin(fmax(q, (double)-hw), (double)(L - 1 - hw));
  return (int8_t)(16 * (int)q);
}

__global__ void k_l8_codes_tok(const double* __restrict__ tok, const uint8_t* __restrict__ mask,
                               int64_t G, int64_t n, int8_t* __restrict__ codes) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= G * 2 * n) return;
  const int64_t pos = idx % n, gt = idx / n;
  int64_t src = idx;
  if ((gt & 1) && !mask[idx]) src = (gt - 1) * n + pos;     // conceal P with the I token
  int8_t q[16] = {0};
  if (mask[src]) {
#pragma unroll
    for (int i = 0; i < kChannels; ++i) q[i] = l8_snap(tok[src * kChannels + i], i);
  }
  *reinterpret_cast<uint4*>(codes + idx * 16) = *reinterpret_cast<const uint4*>(q);
}

__global__ void k_l8_codes_pkt(const uint8_t* __restrict__ buf, const RowInfo* __restrict__ rows,
                               const int32_t* __restrict__ tokoff, int G, int Ht, int Wt,
                               int8_t* __restrict__ codes) {
  const int64_t n = (int64_t)Ht * Wt;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)G * 2 * n) return;
  const int64_t pos = idx % n, gt = idx / n;
  const int y = (int)(pos / Wt), x = (int)(pos % Wt);
  int64_t r = gt * Ht + y;
  int slot = tokoff[r * Wt + x];
  if ((gt & 1) && slot < 0) {                 // conceal with the co-located I token
    r = (gt - 1) * Ht + y;
    slot = tokoff[r * Wt + x];
  }
  int8_t q[16] = {0};
  if (slot >= 0) {
    const RowInfo ri = rows[r];
    const uint8_t* p = buf + ri.payload + (int64_t)slot * kChannels;
#pragma unroll
    for (int i = 0; i < kChannels; ++i) q[i] = l8_snap(ri.qmin + (double)p[i] * ri.step, i);
  }
  *reinterpret_cast<uint4*>(codes + idx * 16) = *reinterpret_cast<const uint4*>(q);
}

// one thread per (token, tap): tap < 18 copies the 12 code bytes of that
// (2,3,3) neighbour (zero outside the frame / before t = 0) to channels
// 12 tap .. 12 tap + 11 as three 4-byte stores; tap 18 zeroes channels 216..255
__global__ void k_l8_gather233(const int8_t* __restrict__ codes, int G, int Ht, int Wt,
                               int8_t* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)Ht * Wt;
  if (e >= (int64_t)G * 2 * n * 19) return;
  const int tap = (int)(e % 19);
  const int64_t tokn = e / 19;
  uint32_t* dst = reinterpret_cast<uint32_t*>(out + tokn * 256);
  if (tap == 18) {
#pragma unroll
    for (int i = 54; i < 64; ++i) dst[i] = 0u;
    return;
  }
  const int64_t pos = tokn % n, gt = tokn / n;
  const int t = (int)(gt & 1);
  const int y = (int)(pos / Wt), x = (int)(pos - (int64_t)y * Wt);
  const int tt = t + tap / 9 - 1, yy = y + (tap / 3) % 3 - 1, xx = x + tap % 3 - 1;
  uint4 v = make_uint4(0, 0, 0, 0);
  if (tt >= 0 && yy >= 0 && yy < Ht && xx >= 0 && xx < Wt)
    v = __ldg(reinterpret_cast<const uint4*>(codes + ((((gt - t + tt) * Ht) + yy) * Wt + xx) * 16));
  dst[tap * 3 + 0] = v.x;
  dst[tap * 3 + 1] = v.y;
  dst[tap * 3 + 2] = v.z;
}

static int l8_gather(const int8_t* codes, int G, int Ht, int Wt, void* out, cudaStream_t st) {
  const int64_t total = (int64_t)G * 2 * Ht * Wt * 19;
  k_l8_gather233<<<(unsigned)ceil_div64(total, 256), 256, 0, st>>>(codes, G, Ht, Wt,
                                                                   static_cast<int8_t*>(out));
  SST_LAUNCH_CHECK();
  return SST_OK;
}

}  // namespace sst

extern "C" int sst_lt8_dec_in(const double* tok, const uint8_t* mask, int G, int Ht, int Wt, void* ws,
                              void* out, void* stream) {
  if (!tok || !mask || !ws || !out || G <= 0 || Ht <= 0 || Wt <= 0) return SST_ERR_ARG;
  if ((reinterpret_cast<uintptr_t>(ws) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
    return SST_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = (int64_t)Ht * Wt;
  k_l8_codes_tok<<<(unsigned)ceil_div64((int64_t)G * 2 * n, 256), 256, 0, st>>>(
      tok, mask, G, n, static_cast<int8_t*>(ws));
  SST_LAUNCH_CHECK();
  return l8_gather(static_cast<const int8_t*>(ws), G, Ht, Wt, out, st);
}

extern "C" int64_t sst_lt8_unpack_workspace(int G, int Ht, int Wt) {
  const int64_t base = (sst_unpack_decode_workspace(G, Ht, Wt) + 15) / 16 * 16;
  return base + 2 * (int64_t)G * Ht * Wt * 16;
}

extern "C" int sst_lt8_unpack_dec_in(const uint8_t* buf, const int64_t* off, SstPacketInfo* info,
                                     const int32_t* target, int64_t n, int G, int Ht, int Wt,
                                     const uint32_t* exp_gop, uint32_t* winner, int32_t* stats,
                                     void* ws, void* out, void* stream) {
  if (n < 0 || G < 0 || Ht <= 0 || Wt <= 0) return SST_ERR_ARG;
  if (G == 0) return SST_OK;
  if (!exp_gop || !winner || !stats || !out || !ws) return SST_ERR_ARG;
  if (n > 0 && (!buf || !off || !info || !target)) return SST_ERR_ARG;
  if (Ht > 65535 || G > 65535) return SST_ERR_ARG;
  if ((reinterpret_cast<uintptr_t>(ws) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
    return SST_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = route_packets(info, target, n, 2 * G, Ht, nullptr, exp_gop, winner, stats, st);
  if (rc != SST_OK) return rc;
  const int64_t nrows = 2 * (int64_t)G * Ht;
  RowInfo* rows = static_cast<RowInfo*>(ws);
  int32_t* tokoff = reinterpret_cast<int32_t*>(rows + nrows);
  int8_t* codes = static_cast<int8_t*>(ws) + (sst_unpack_decode_workspace(G, Ht, Wt) + 15) / 16 * 16;
  k_rowprep<<<(unsigned)ceil_div64(nrows, 8), 256, 0, st>>>(off, info, buf, winner, nrows, Ht, Wt,
                                                            rows, tokoff, stats);
  SST_LAUNCH_CHECK();
  const int64_t total = nrows * Wt;
  k_l8_codes_pkt<<<(unsigned)ceil_div64(total, 256), 256, 0, st>>>(buf, rows, tokoff, G, Ht, Wt,
                                                                   codes);
  SST_LAUNCH_CHECK();
  return l8_gather(codes, G, Ht, Wt, out, st);
}
