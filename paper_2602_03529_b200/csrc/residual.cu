// Residual enhancement layer and its adaptive range coder
// (§8 f2).
//
//   k_residual      compute_residual + aggregate_residual + sparsify_quantize
//                   (residual.py:62-105): per working-resolution sample, the
//                   float64 temporal mean of x(t) - x_hat(t) (sequential sum
//                   from 0.0, / 9), rint-quantised to int16 on the 1/127 grid
//                   and thresholded; also the |avg| ranking key used by
//                   fit_to_budget and the kept-entry count.
//   k_apply_residual apply_residual (residual.py:108-127) on the two unique
//                   reconstructions (I frame, shared P frame).
//   k_rc_encode / k_rc_decode
//                   rangecoder.py:75-243: zero-run symbolisation, order-0
//                   adaptive model (counts start at 1, halved at total 2^16)
//                   and the carry-less 32-bit range coder.  The coder is
//                   serial per stream (adaptive model), so one CTA owns one
//                   stream: all its threads first compact the non-zero
//                   positions of the scan (ballot/popc, index order), then one
//                   thread codes them with a Fenwick tree for the cumulative
//                   frequencies (O(log 510) instead of the reference's O(510)).
#include <climits>
#include <cstdlib>

#include "common.cuh"

namespace sst {

// ---------------------------------------------------------------------------
// residual

__global__ void k_residual(const float* __restrict__ work, const float* __restrict__ img,
                           int64_t n, double theta, double step, double* __restrict__ avg_out,
                           int16_t* __restrict__ dense, double* __restrict__ mags,
                           int32_t* __restrict__ count) {
  // grid.y = GoP
  const int g = blockIdx.y;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool kept = false;
  if (e < n) {
    const float* x = work + (int64_t)g * kGop * n;
    const double ii = (double)img[(int64_t)g * 2 * n + e];
    const double pp = (double)img[((int64_t)g * 2 + 1) * n + e];
    double acc = 0.0 + ((double)x[e] - ii);                 // frame 0 vs I reconstruction
#pragma unroll
    for (int t = 1; t < kGop; ++t) acc = acc + ((double)x[(int64_t)t * n + e] - pp);
    const double avg = acc / 9.0;
    if (avg_out) avg_out[(int64_t)g * n + e] = avg;
    double q = rint(avg / step);
    q = q < -127.0 ? -127.0 : (q > 127.0 ? 127.0 : q);
    const int16_t qv = (int16_t)(int)q;
    const double mag = fabs(avg);
    const int aq = qv < 0 ? -qv : qv;
    kept = mag >= theta && qv != 0 && (double)aq * step >= theta;
    dense[(int64_t)g * n + e] = kept ? qv : (int16_t)0;
    if (mags) mags[(int64_t)g * n + e] = kept ? mag : -1.0;
  }
  const unsigned bal = __ballot_sync(0xffffffffu, kept);
  if ((threadIdx.x & 31) == 0 && bal) atomicAdd(&count[g], __popc(bal));
}

// aggregate_residual: mean over the window axis, sequential from 0.0, / T
// (residual.py:76-83 -> numpy add.reduce over axis 0, then true_divide)
__global__ void k_mean_axis0(const double* __restrict__ res, int T, int64_t n,
                             double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double acc = 0.0 + res[e];
  for (int t = 1; t < T; ++t) acc = acc + res[(int64_t)t * n + e];
  out[e] = acc / (double)T;
}

// sparsify_quantize from a given float64 average (residual.py:86-105)
__global__ void k_sparsify(const double* __restrict__ avg, int64_t n, double theta, double step,
                           int16_t* __restrict__ dense, double* __restrict__ mags,
                           int32_t* __restrict__ count) {
  const int g = blockIdx.y;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool kept = false;
  if (e < n) {
    const double a = avg[(int64_t)g * n + e];
    double q = rint(a / step);
    q = q < -127.0 ? -127.0 : (q > 127.0 ? 127.0 : q);
    const int16_t qv = (int16_t)(int)q;
    const double mag = fabs(a);
    const int aq = qv < 0 ? -qv : qv;
    kept = mag >= theta && qv != 0 && (double)aq * step >= theta;
    dense[(int64_t)g * n + e] = kept ? qv : (int16_t)0;
    if (mags) mags[(int64_t)g * n + e] = kept ? mag : -1.0;
  }
  const unsigned bal = __ballot_sync(0xffffffffu, kept);
  if ((threadIdx.x & 31) == 0 && bal) atomicAdd(&count[g], __popc(bal));
}

__global__ void k_apply_residual(float* __restrict__ img, const int16_t* __restrict__ dense,
                                 const int32_t* __restrict__ count, int64_t n, double step) {
  const int g = blockIdx.y;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n || count[g] == 0) return;           // empty residual: recon unchanged
  const double delta = (double)dense[(int64_t)g * n + e] * step;
#pragma unroll
  for (int im = 0; im < 2; ++im) {
    float* p = img + ((int64_t)g * 2 + im) * n + e;
    *p = (float)clip01((double)*p + delta);
  }
}

// keep only the chosen entries of a dense scan (fit_to_budget candidates)
__global__ void k_mask_scan(const int16_t* __restrict__ dense, const uint8_t* __restrict__ keep,
                            int64_t total, int16_t* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < total) out[e] = keep[e] ? dense[e] : (int16_t)0;
}

// ---------------------------------------------------------------------------
// range coder

constexpr int kAlpha = 510;
constexpr int kFen = 512;                         // Fenwick size (power of two >= 510)
constexpr uint64_t kMask32 = 0xFFFFFFFFull;
constexpr uint64_t kTop = 1ull << 24;
constexpr uint64_t kBottom = 1ull << 16;
constexpr int kRcThreads = 1024;

struct Model {
  uint32_t fen[kFen + 1];                         // 1-based Fenwick tree of counts
  uint32_t cnt[kFen];
  uint32_t total;
};

__device__ void model_build(Model& m) {
  for (int i = 0; i <= kFen; ++i) m.fen[i] = 0;
  uint32_t tot = 0;
  for (int s = 0; s < kAlpha; ++s) {
    tot += m.cnt[s];
    for (int i = s + 1; i <= kFen; i += i & -i) m.fen[i] += m.cnt[s];
  }
  m.total = tot;
}

__device__ __forceinline__ uint32_t model_cum(const Model& m, int s) {   // sum cnt[0..s)
  uint32_t c = 0;
  for (int i = s; i > 0; i -= i & -i) c += m.fen[i];
  return c;
}

__device__ __forceinline__ void model_update(Model& m, int s) {
  m.cnt[s] += 1;
  for (int i = s + 1; i <= kFen; i += i & -i) m.fen[i] += 1;
  m.total += 1;
  if (m.total >= (uint32_t)kBottom) {              // rangecoder.py:147-149
    for (int t = 0; t < kAlpha; ++t) m.cnt[t] = (m.cnt[t] + 1) / 2;
    model_build(m);
  }
}

// largest symbol whose cumulative low is <= target; returns its low in *lo
__device__ __forceinline__ int model_find(const Model& m, uint32_t target, uint32_t* lo) {
  int pos = 0;
  uint32_t acc = 0;
  for (int step = kFen; step > 0; step >>= 1) {
    const int nxt = pos + step;
    if (nxt <= kFen && acc + m.fen[nxt] <= target) {
      pos = nxt;
      acc += m.fen[nxt];
    }
  }
  *lo = acc;
  return pos;                                      // symbol index (0-based) = pos
}

struct Enc {
  uint64_t low, range;
  uint8_t* out;
  int64_t pos, cap;
  bool overflow;
};

__device__ __forceinline__ void enc_symbol(Enc& e, Model& m, int sym) {
  const uint64_t c = model_cum(m, sym);
  const uint64_t d = c + m.cnt[sym];
  // range < 2^32 and total < 2^16: a 32-bit division gives the same quotient
  // as the reference's arbitrary-precision one at a fraction of the cost of
  // the 64-bit software division
  const uint64_t r = (uint64_t)((uint32_t)e.range / m.total);
  e.low += c * r;
  e.range = (d - c) * r;
  while ((e.low ^ (e.low + e.range)) < kTop || e.range < kBottom) {
    if ((e.low ^ (e.low + e.range)) >= kTop) e.range = (kMask32 + 1 - e.low) & (kBottom - 1);
    if (e.pos < e.cap) e.out[e.pos] = (uint8_t)((e.low >> 24) & 0xFF);
    else e.overflow = true;
    e.pos += 1;
    e.low = (e.low << 8) & kMask32;
    e.range <<= 8;
  }
  model_update(m, sym);
}

// Compact the non-zero positions of one stream's scan into idx (index order);
// returns their count.  All threads of the CTA.
__device__ int64_t compact_nonzero(const int16_t* scan, int64_t n, int64_t* idx, int* s_warp,
                                   int64_t* s_base) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) *s_base = 0;
  __syncthreads();
  for (int64_t b = 0; b < n; b += kRcThreads) {
    const int64_t j = b + tid;
    const bool nz = j < n && scan[j] != 0;
    const unsigned bal = __ballot_sync(0xffffffffu, nz);
    if (lane == 0) s_warp[wid] = __popc(bal);
    __syncthreads();
    int off = 0;
    for (int w = 0; w < wid; ++w) off += s_warp[w];
    const int64_t base = *s_base;
    if (nz) idx[base + off + __popc(bal & ((1u << lane) - 1u))] = j;
    __syncthreads();
    if (tid == 0) {
      int tot = 0;
      for (int w = 0; w < kRcThreads / 32; ++w) tot += s_warp[w];
      *s_base = base + tot;
    }
    __syncthreads();
  }
  return *s_base;
}

// One CTA per stream: encode_scan(scan[g]) -> out[g*cap ...], len[g]
// (len = -1 if the output would exceed cap).
__global__ void __launch_bounds__(kRcThreads)
    k_rc_encode(const int16_t* __restrict__ scans, int64_t n, int64_t* __restrict__ idx_ws,
                uint8_t* __restrict__ out, int64_t cap, int64_t* __restrict__ out_len) {
  __shared__ Model m;
  __shared__ int s_warp[kRcThreads / 32];
  __shared__ int64_t s_base;
  const int g = blockIdx.x;
  const int16_t* scan = scans + (int64_t)g * n;
  int64_t* idx = idx_ws + (int64_t)g * n;
  const int64_t nnz = compact_nonzero(scan, n, idx, s_warp, &s_base);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kFen; ++s) m.cnt[s] = s < kAlpha ? 1u : 0u;
  model_build(m);
  Enc e{0, kMask32, out + (int64_t)g * cap, 0, cap, false};
  int64_t pos = 0;
  for (int64_t i = 0; i < nnz; ++i) {              // rangecoder.py:75-94
    const int64_t j = idx[i];
    int64_t gap = j - pos;
    while (gap > 255) {
      enc_symbol(e, m, 255);
      gap -= 255;
    }
    if (gap) enc_symbol(e, m, (int)gap);
    const int v = scan[j];
    enc_symbol(e, m, v < 0 ? v + 383 : v + 382);
    pos = j + 1;
  }
  enc_symbol(e, m, 0);                              // EOS
  for (int k = 0; k < 4; ++k) {                     // rangecoder.py:182-184
    if (e.pos < e.cap) e.out[e.pos] = (uint8_t)((e.low >> 24) & 0xFF);
    else e.overflow = true;
    e.pos += 1;
    e.low = (e.low << 8) & kMask32;
  }
  out_len[g] = e.overflow ? -e.pos : e.pos;
}

// One CTA per stream: decode_scan(data[g], n) -> scan[g]; status[g]:
// 0 ok, 1 truncated, 2 zero run overruns, 3 value overruns, 4 symbol budget
__global__ void __launch_bounds__(kRcThreads)
    k_rc_decode(const uint8_t* __restrict__ data, const int64_t* __restrict__ off,
                const int64_t* __restrict__ len, int64_t n, int16_t* __restrict__ scans,
                int32_t* __restrict__ status) {
  __shared__ Model m;
  const int g = blockIdx.x;
  int16_t* scan = scans + (int64_t)g * n;
  for (int64_t j = threadIdx.x; j < n; j += kRcThreads) scan[j] = 0;
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint8_t* src = data + off[g];
  const int64_t nb = len[g];
  int64_t p = 0;
  int st = 0;
  for (int s = 0; s < kFen; ++s) m.cnt[s] = s < kAlpha ? 1u : 0u;
  model_build(m);
  uint64_t state = 0;
  for (int k = 0; k < 4; ++k) {
    if (p >= nb) { st = 1; break; }
    state = (state << 8) | src[p++];
  }
  uint64_t low = 0, range = kMask32;
  int64_t pos = 0, nsym = 0;
  while (st == 0) {
    const uint64_t total = m.total;
    const uint64_t r = (uint64_t)((uint32_t)range / (uint32_t)total);   // range < 2^32
    const uint64_t diff = state - low;
    uint64_t val = (diff >> 32) == 0 ? (uint64_t)((uint32_t)diff / (uint32_t)r)
                                     : diff / r;   // rangecoder.py:217-219 (wrapped: 64-bit)
    if (val >= total) val = total - 1;
    uint32_t c32;
    const int sym = model_find(m, (uint32_t)val, &c32);
    const uint64_t c = c32, d = c + m.cnt[sym];
    low += c * r;
    range = (d - c) * r;
    while ((low ^ (low + range)) < kTop || range < kBottom) {
      if ((low ^ (low + range)) >= kTop) range = (kMask32 + 1 - low) & (kBottom - 1);
      if (p >= nb) { st = 1; break; }
      state = ((state << 8) | src[p++]) & kMask32;
      low = (low << 8) & kMask32;
      range <<= 8;
    }
    if (st) break;
    model_update(m, sym);
    ++nsym;
    if (sym == 0) break;                            // EOS
    if (sym <= 255) {                               // zero run (rangecoder.py:107-110)
      pos += sym;
      if (pos > n) { st = 2; break; }
    } else {
      if (pos >= n) { st = 3; break; }
      scan[pos++] = (int16_t)(sym <= 382 ? sym - 383 : sym - 382);
    }
    if (nsym >= (1 << 24)) { st = 4; break; }
  }
  status[g] = st;
}

// ---- warp-cooperative coder -------------------------------------------------
// The same adaptive model and coder, but the model lives in the registers of
// one warp: lane l owns the counts of symbols 16l .. 16l+15.  cum(s) is a warp
// sum of per-lane partials (5 shuffles), the decoder's symbol search a warp
// prefix scan + ballot, the halving is lane-parallel; the coder state is kept
// uniform across the warp (every lane runs the same arithmetic), lane 0 writes.
struct WarpModel {
  uint32_t c[16];
  uint32_t lsum;
  uint32_t total;
};

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void wm_init(WarpModel& m, int lane) {
  m.lsum = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    m.c[k] = (16 * lane + k) < kAlpha ? 1u : 0u;
    m.lsum += m.c[k];
  }
  m.total = warp_sum_u32(m.lsum);
}

__device__ __forceinline__ void wm_lookup(const WarpModel& m, int lane, int sym, uint32_t& cum,
                                          uint32_t& cnt) {
  const int owner = sym >> 4, off = sym & 15;
  uint32_t part = 0, mine = 0;
  if (lane < owner) {
    part = m.lsum;
  } else if (lane == owner) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (k < off) part += m.c[k];
      if (k == off) mine = m.c[k];
    }
  }
  cum = warp_sum_u32(part);
  cnt = __shfl_sync(0xffffffffu, mine, owner);
}

__device__ __forceinline__ void wm_update(WarpModel& m, int lane, int sym) {
  const int owner = sym >> 4, off = sym & 15;
  if (lane == owner) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (k == off) m.c[k] += 1;
    m.lsum += 1;
  }
  m.total += 1;
  if (m.total >= (uint32_t)kBottom) {               // rangecoder.py:147-149
    m.lsum = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      m.c[k] = (m.c[k] + 1) / 2;                    // 0 stays 0 for s >= 510
      m.lsum += m.c[k];
    }
    m.total = warp_sum_u32(m.lsum);
  }
}

struct WEnc {
  uint64_t low, range;
  int64_t pos;
};

__device__ __forceinline__ void wenc_symbol(WEnc& e, WarpModel& m, int lane, int sym,
                                            uint8_t* out, int64_t cap) {
  uint32_t c32, n32;
  wm_lookup(m, lane, sym, c32, n32);
  const uint64_t r = (uint64_t)((uint32_t)e.range / m.total);
  e.low += (uint64_t)c32 * r;
  e.range = (uint64_t)n32 * r;
  while ((e.low ^ (e.low + e.range)) < kTop || e.range < kBottom) {
    if ((e.low ^ (e.low + e.range)) >= kTop) e.range = (kMask32 + 1 - e.low) & (kBottom - 1);
    if (lane == 0 && e.pos < cap) out[e.pos] = (uint8_t)((e.low >> 24) & 0xFF);
    e.pos += 1;
    e.low = (e.low << 8) & kMask32;
    e.range <<= 8;
  }
  wm_update(m, lane, sym);
}

__global__ void __launch_bounds__(kRcThreads)
    k_rc_encode_w(const int16_t* __restrict__ scans, int64_t n, int64_t* __restrict__ idx_ws,
                  uint8_t* __restrict__ out, int64_t cap, int64_t* __restrict__ out_len) {
  __shared__ int s_warp[kRcThreads / 32];
  __shared__ int64_t s_base;
  const int g = blockIdx.x;
  const int16_t* scan = scans + (int64_t)g * n;
  int64_t* idx = idx_ws + (int64_t)g * n;
  const int64_t nnz = compact_nonzero(scan, n, idx, s_warp, &s_base);
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  WarpModel m;
  wm_init(m, lane);
  uint8_t* o = out + (int64_t)g * cap;
  WEnc e{0, kMask32, 0};
  int64_t pos = 0;
  // the non-zero positions and values are fetched 32 at a time (one per lane,
  // coalesced) and handed to the serial coder by shuffles, so the coder never
  // waits on a dependent global load
  for (int64_t base = 0; base < nnz; base += 32) {
    const int64_t ii = base + lane;
    const int64_t jl = ii < nnz ? idx[ii] : 0;
    const int vl = ii < nnz ? (int)scan[jl] : 0;
    const int nb32 = (int)min((int64_t)32, nnz - base);
    for (int t = 0; t < nb32; ++t) {                // rangecoder.py:75-94
      const int64_t j = __shfl_sync(0xffffffffu, jl, t);
      const int v = __shfl_sync(0xffffffffu, vl, t);
      int64_t gap = j - pos;
      while (gap > 255) {
        wenc_symbol(e, m, lane, 255, o, cap);
        gap -= 255;
      }
      if (gap) wenc_symbol(e, m, lane, (int)gap, o, cap);
      wenc_symbol(e, m, lane, v < 0 ? v + 383 : v + 382, o, cap);
      pos = j + 1;
    }
  }
  wenc_symbol(e, m, lane, 0, o, cap);                // EOS
  for (int k = 0; k < 4; ++k) {                      // rangecoder.py:182-184
    if (lane == 0 && e.pos < cap) o[e.pos] = (uint8_t)((e.low >> 24) & 0xFF);
    e.pos += 1;
    e.low = (e.low << 8) & kMask32;
  }
  if (lane == 0) out_len[g] = e.pos > cap ? -e.pos : e.pos;
}

__global__ void __launch_bounds__(kRcThreads)
    k_rc_decode_w(const uint8_t* __restrict__ data, const int64_t* __restrict__ off,
                  const int64_t* __restrict__ len, int64_t n, int16_t* __restrict__ scans,
                  int32_t* __restrict__ status) {
  const int g = blockIdx.x;
  int16_t* scan = scans + (int64_t)g * n;
  for (int64_t j = threadIdx.x; j < n; j += kRcThreads) scan[j] = 0;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const uint8_t* src = data + off[g];
  const int64_t nb = len[g];
  int64_t p = 0;
  int st = 0;
  WarpModel m;
  wm_init(m, lane);
  // 32-byte window of the payload held one byte per lane (coalesced refill)
  int64_t wbase = 0;
  uint32_t wbyte = lane < nb ? src[lane] : 0;
  auto next_byte = [&]() -> uint32_t {
    if (p - wbase >= 32) {
      wbase = p;
      wbyte = wbase + lane < nb ? src[wbase + lane] : 0;
    }
    const uint32_t b = __shfl_sync(0xffffffffu, wbyte, (int)(p - wbase));
    ++p;
    return b;
  };
  uint64_t state = 0;
  for (int k = 0; k < 4; ++k) {
    if (p >= nb) { st = 1; break; }
    state = (state << 8) | next_byte();
  }
  uint64_t low = 0, range = kMask32;
  int64_t pos = 0, nsym = 0;
  while (st == 0) {
    const uint64_t total = m.total;
    const uint64_t r = (uint64_t)((uint32_t)range / (uint32_t)total);
    const uint64_t diff = state - low;
    uint64_t val = (diff >> 32) == 0 ? (uint64_t)((uint32_t)diff / (uint32_t)r) : diff / r;
    if (val >= total) val = total - 1;
    // symbol search: lane prefix sums, then the owner lane scans its 16 counts
    uint32_t incl = m.lsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const uint32_t excl = incl - m.lsum;
    const unsigned bal = __ballot_sync(0xffffffffu, (uint64_t)excl <= val);
    const int owner = 31 - __clz(bal);
    int soff = 0;
    uint32_t lo = 0, cnt = 0;
    if (lane == owner) {
      uint32_t acc = excl;
      bool found = false;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (!found && (uint64_t)(acc + m.c[k]) > val) {
          found = true;
          soff = k;
          lo = acc;
          cnt = m.c[k];
        }
        acc += m.c[k];
      }
    }
    soff = __shfl_sync(0xffffffffu, soff, owner);
    lo = __shfl_sync(0xffffffffu, lo, owner);
    cnt = __shfl_sync(0xffffffffu, cnt, owner);
    const int sym = owner * 16 + soff;
    low += (uint64_t)lo * r;
    range = (uint64_t)cnt * r;
    while ((low ^ (low + range)) < kTop || range < kBottom) {
      if ((low ^ (low + range)) >= kTop) range = (kMask32 + 1 - low) & (kBottom - 1);
      if (p >= nb) { st = 1; break; }
      state = ((state << 8) | next_byte()) & kMask32;
      low = (low << 8) & kMask32;
      range <<= 8;
    }
    if (st) break;
    wm_update(m, lane, sym);
    ++nsym;
    if (sym == 0) break;                            // EOS
    if (sym <= 255) {                               // zero run (rangecoder.py:107-110)
      pos += sym;
      if (pos > n) { st = 2; break; }
    } else {
      if (pos >= n) { st = 3; break; }
      if (lane == 0) scan[pos] = (int16_t)(sym <= 382 ? sym - 383 : sym - 382);
      ++pos;
    }
    if (nsym >= (1 << 24)) { st = 4; break; }
  }
  if (lane == 0) status[g] = st;
}

// Chunked compaction for the cumulative-table coder (NT threads): thread t
// counts the non-zeros of its contiguous chunk, one block scan places the
// chunks, and a second pass writes the indices -- two barriers in total
// instead of three per NT elements.
template <int NT>
__device__ int64_t compact_nonzero_chunked(const int16_t* scan, int64_t n, int64_t* idx,
                                           int64_t* s_part) {
  const int tid = threadIdx.x;
  const int64_t chunk = (n + NT - 1) / NT;
  const int64_t b0 = min(n, (int64_t)tid * chunk), b1 = min(n, b0 + chunk);
  int64_t cnt = 0;
  for (int64_t j = b0; j < b1; ++j) cnt += scan[j] != 0;
  s_part[tid] = cnt;
  __syncthreads();
  if (tid == 0) {                     // exclusive scan of NT chunk counts
    int64_t run = 0;
    for (int i = 0; i < NT; ++i) {
      const int64_t c = s_part[i];
      s_part[i] = run;
      run += c;
    }
    s_part[NT] = run;
  }
  __syncthreads();
  int64_t o = s_part[tid];
  for (int64_t j = b0; j < b1; ++j)
    if (scan[j] != 0) idx[o++] = j;
  __syncthreads();
  return s_part[NT];
}

constexpr int kRcThreadsC = 256;

// ---- cumulative-table coder (default) --------------------------------------
// The same adaptive model held by one warp as a CUMULATIVE table: lane l keeps,
// for its symbols s = 16l + k, the count cnt[k] and the exclusive prefix
// cum[k] = sum of the counts of all symbols below s.  A symbol's (cum, cnt)
// is then one register select in every lane plus ONE packed shuffle from its
// owner (cum, cnt < 2^16 while total < 2^16), the decoder's search one ballot
// (cum is strictly increasing: every live count is >= 1) plus one shuffle,
// and the update 16 predicated adds per lane with no cross-lane dependency --
// instead of a 5-shuffle warp reduction (encode) or scan (decode) per symbol.
// The rare halving (rangecoder.py:147-149) rebuilds cum with one warp scan.
struct CumModel {
  uint32_t pc[16];                                 // (cum << 16) | cnt of symbol 16 lane + k
  uint32_t total;
};

__device__ __forceinline__ void cm_rebuild(CumModel& m, int lane, const uint32_t (&cnt)[16]) {
  uint32_t local = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) local += cnt[k];
  uint32_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  uint32_t run = incl - local;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    m.pc[k] = (run << 16) | cnt[k];
    run += cnt[k];
  }
  m.total = __shfl_sync(0xffffffffu, incl, 31);
}

__device__ __forceinline__ void cm_init(CumModel& m, int lane) {
  uint32_t cnt[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) cnt[k] = (16 * lane + k) < kAlpha ? 1u : 0u;
  cm_rebuild(m, lane, cnt);
}

// a[idx] for idx in [0, 16) as a depth-4 select tree (a linear select chain
// would put 16 dependent SELs on the coder's serial path)
__device__ __forceinline__ uint32_t sel16(const uint32_t (&a)[16], int idx) {
  uint32_t b[8], c[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) b[i] = (idx & 1) ? a[2 * i + 1] : a[2 * i];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i] = (idx & 2) ? b[2 * i + 1] : b[2 * i];
  const uint32_t d0 = (idx & 4) ? c[1] : c[0], d1 = (idx & 4) ? c[3] : c[2];
  return (idx & 8) ? d1 : d0;
}

// (cum << 16) | cnt of symbol `sym` on every lane
__device__ __forceinline__ uint32_t cm_lookup(const CumModel& m, int sym) {
  return __shfl_sync(0xffffffffu, sel16(m.pc, sym & 15), sym >> 4);
}

__device__ __forceinline__ void cm_update(CumModel& m, int lane, int sym) {
  // symbols above sym gain 1 in cum, sym itself 1 in cnt: one 32-bit mask
  // holds both (bit k: symbol 16 lane + k is sym; bit 16 + k: it lies above),
  // so each of the 16 entries costs a shift, an AND and an add
  const int rc = min(max(sym - 16 * lane, -1), 16);
  const uint32_t above = (0xFFFFu << (rc + 1)) & 0xFFFFu;
  const uint32_t mine = (unsigned)rc < 16u ? 1u << rc : 0u;
  const uint32_t inc = (above << 16) | mine;
#pragma unroll
  for (int k = 0; k < 16; ++k) m.pc[k] += (inc >> k) & 0x10001u;
  m.total += 1;
  if (m.total >= (uint32_t)kBottom) {               // rangecoder.py:147-149
    uint32_t cnt[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) cnt[k] = ((m.pc[k] & 0xFFFFu) + 1) / 2;   // 0 stays 0 (s >= 510)
    cm_rebuild(m, lane, cnt);
  }
}

// floor(a / b) for b >= 1 through a float reciprocal, corrected to exact
__device__ __forceinline__ uint32_t udiv32(uint32_t a, uint32_t b) {
  uint32_t q = __float2uint_rz(__fdividef((float)a, (float)b));
  const int64_t r = (int64_t)a - (int64_t)q * b;
  if (r < 0) q -= (uint32_t)((-r + b - 1) / b);   // rare: the estimate overshot
  else if (r >= (int64_t)b) q += (uint32_t)(r / b);
  return q;
}

__device__ __forceinline__ void cenc_symbol(WEnc& e, CumModel& m, int lane, int sym, uint8_t* out,
                                            int64_t cap) {
  const uint32_t cc = cm_lookup(m, sym);
  const uint64_t r = (uint64_t)udiv32((uint32_t)e.range, m.total);
  e.low += (uint64_t)(cc >> 16) * r;
  e.range = (uint64_t)(cc & 0xFFFFu) * r;
  while ((e.low ^ (e.low + e.range)) < kTop || e.range < kBottom) {
    if ((e.low ^ (e.low + e.range)) >= kTop) e.range = (kMask32 + 1 - e.low) & (kBottom - 1);
    if (lane == 0 && e.pos < cap) out[e.pos] = (uint8_t)((e.low >> 24) & 0xFF);
    e.pos += 1;
    e.low = (e.low << 8) & kMask32;
    e.range <<= 8;
  }
  cm_update(m, lane, sym);
}

__global__ void __launch_bounds__(kRcThreadsC, 1)
    k_rc_encode_c(const int16_t* __restrict__ scans, int64_t n, int64_t* __restrict__ idx_ws,
                  uint8_t* __restrict__ out, int64_t cap, int64_t* __restrict__ out_len) {
  __shared__ int64_t s_part[kRcThreadsC + 1];
  const int g = blockIdx.x;
  const int16_t* scan = scans + (int64_t)g * n;
  int64_t* idx = idx_ws + (int64_t)g * n;
  const int64_t nnz = compact_nonzero_chunked<kRcThreadsC>(scan, n, idx, s_part);
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  CumModel m;
  cm_init(m, lane);
  uint8_t* o = out + (int64_t)g * cap;
  WEnc e{0, kMask32, 0};
  int64_t pos = 0;
  for (int64_t base = 0; base < nnz; base += 32) {
    const int64_t ii = base + lane;
    const int64_t jl = ii < nnz ? idx[ii] : 0;
    const int vl = ii < nnz ? (int)scan[jl] : 0;
    const int nb32 = (int)min((int64_t)32, nnz - base);
    for (int t = 0; t < nb32; ++t) {                // rangecoder.py:75-94
      const int64_t j = __shfl_sync(0xffffffffu, jl, t);
      const int v = __shfl_sync(0xffffffffu, vl, t);
      int64_t gap = j - pos;
      while (gap > 255) {
        cenc_symbol(e, m, lane, 255, o, cap);
        gap -= 255;
      }
      if (gap) cenc_symbol(e, m, lane, (int)gap, o, cap);
      cenc_symbol(e, m, lane, v < 0 ? v + 383 : v + 382, o, cap);
      pos = j + 1;
    }
  }
  cenc_symbol(e, m, lane, 0, o, cap);                // EOS
  for (int k = 0; k < 4; ++k) {                      // rangecoder.py:182-184
    if (lane == 0 && e.pos < cap) o[e.pos] = (uint8_t)((e.low >> 24) & 0xFF);
    e.pos += 1;
    e.low = (e.low << 8) & kMask32;
  }
  if (lane == 0) out_len[g] = e.pos > cap ? -e.pos : e.pos;
}

template <bool kFloatQ>
__global__ void __launch_bounds__(kRcThreadsC, 1)
    k_rc_decode_c(const uint8_t* __restrict__ data, const int64_t* __restrict__ off,
                  const int64_t* __restrict__ len, int64_t n, int16_t* __restrict__ scans,
                  int32_t* __restrict__ status) {
  const int g = blockIdx.x;
  int16_t* scan = scans + (int64_t)g * n;
  for (int64_t j = threadIdx.x; j < n; j += kRcThreadsC) scan[j] = 0;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const uint8_t* src = data + off[g];
  const int64_t nb = len[g];
  int64_t p = 0;
  int st = 0;
  CumModel m;
  cm_init(m, lane);
  int64_t wbase = 0;
  uint32_t wbyte = lane < nb ? src[lane] : 0;
  auto next_byte = [&]() -> uint32_t {
    if (p - wbase >= 32) {
      wbase = p;
      wbyte = wbase + lane < nb ? src[wbase + lane] : 0;
    }
    const uint32_t b = __shfl_sync(0xffffffffu, wbyte, (int)(p - wbase));
    ++p;
    return b;
  };
  uint64_t state = 0;
  for (int k = 0; k < 4; ++k) {
    if (p >= nb) { st = 1; break; }
    state = (state << 8) | next_byte();
  }
  uint64_t low = 0, range = kMask32;
  int64_t pos = 0, nsym = 0;
  while (st == 0) {
    const uint32_t total = m.total;
    const uint64_t r = (uint64_t)udiv32((uint32_t)range, total);
    // the symbol is the last one with cum * r <= min(diff, total r - 1), i.e.
    // cum <= min(floor(diff / r), total - 1) (rangecoder.py:216-221) -- no
    // division: every product is <= total r <= range < 2^32, so each lane
    // compares its 16 cumulative counts in 32-bit arithmetic (measured faster
    // than a float quotient estimate plus correction on this serial path)
    const uint64_t diff = state - low;
    const uint32_t tr = total * (uint32_t)r;
    const uint32_t d32 = diff < (uint64_t)tr ? (uint32_t)diff : tr - 1;
    const uint32_t r32 = (uint32_t)r;
    uint32_t le[16];
    if (kFloatQ) {
      // A/B: val = floor(d32 / r) from an approximate float quotient (< 2^16,
      // error < 0.05) corrected once, then 16 packed compares
      uint32_t val = __float2uint_rz(__fdividef(__uint2float_rn(d32), __uint2float_rn(r32)));
      const uint32_t vr = val * r32;
      if (vr > d32) val -= 1;
      else if (d32 - vr >= r32) val += 1;
      const uint32_t vk = (val << 16) | 0xFFFFu;
#pragma unroll
      for (int k = 0; k < 16; ++k) le[k] = m.pc[k] <= vk ? 1u : 0u;
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k) le[k] = (m.pc[k] >> 16) * r32 <= d32 ? 1u : 0u;
    }
    // owner = last lane whose first symbol qualifies; cum is non-decreasing,
    // so the qualifying symbols of a lane are a prefix: offset = count - 1
    const unsigned bal = __ballot_sync(0xffffffffu, le[0] != 0);
    const int owner = 31 - __clz(bal);
    uint32_t s8[8], s4[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s8[i] = le[2 * i] + le[2 * i + 1];
#pragma unroll
    for (int i = 0; i < 4; ++i) s4[i] = s8[2 * i] + s8[2 * i + 1];
    const uint32_t nle = (s4[0] + s4[1]) + (s4[2] + s4[3]);
    const int kl = nle > 0 ? (int)nle - 1 : 0;
    const uint32_t pk = __shfl_sync(0xffffffffu, sel16(m.pc, kl), owner);
    const uint32_t kk = (uint32_t)__shfl_sync(0xffffffffu, kl, owner);
    const int sym = owner * 16 + (int)kk;
    const uint32_t cumv = pk >> 16, cntv = pk & 0xFFFFu;
    low += (uint64_t)cumv * r;
    range = (uint64_t)cntv * r;
    while ((low ^ (low + range)) < kTop || range < kBottom) {
      if ((low ^ (low + range)) >= kTop) range = (kMask32 + 1 - low) & (kBottom - 1);
      if (p >= nb) { st = 1; break; }
      state = ((state << 8) | next_byte()) & kMask32;
      low = (low << 8) & kMask32;
      range <<= 8;
    }
    if (st) break;
    cm_update(m, lane, sym);
    ++nsym;
    if (sym == 0) break;                            // EOS
    if (sym <= 255) {                               // zero run (rangecoder.py:107-110)
      pos += sym;
      if (pos > n) { st = 2; break; }
    } else {
      if (pos >= n) { st = 3; break; }
      if (lane == 0) scan[pos] = (int16_t)(sym <= 382 ? sym - 383 : sym - 382);
      ++pos;
    }
    if (nsym >= (1 << 24)) { st = 4; break; }
  }
  if (lane == 0) status[g] = st;
}

// sum of 16 small values as a 3-input add tree (depth 3, not a 16-long chain)
// (the values pass through an empty asm so the compiler cannot turn the tree
// of 0/1 adds back into a chain of 16 conditional increments)
__device__ __forceinline__ uint32_t sum16(uint32_t (&b)[16]) {
#pragma unroll
  for (int k = 0; k < 16; ++k) asm("" : "+r"(b[k]));
  const uint32_t a0 = b[0] + b[1] + b[2], a1 = b[3] + b[4] + b[5], a2 = b[6] + b[7] + b[8];
  const uint32_t a3 = b[9] + b[10] + b[11], a4 = b[12] + b[13] + b[14];
  return (a0 + a1 + a2) + (a3 + a4 + b[15]);
}

// ---- decoder with a split cumulative table (default) --------------------------
// One warp per CTA (one stream); lane l holds the exclusive cumulative counts
// cum[k] of symbols 16 l + k and `end` = the cumulative count of symbol
// 16 l + 16, so a symbol's count is the difference of two neighbours.  The
// serial chain per symbol is kept short and the instruction count low:
//  * r = range / total: one multiply-high by floor(2^32 / total), fetched from
//    the lane that holds it one symbol ahead (total grows by one per symbol
//    between halvings), plus one correction;
//  * the search: 16 signed IMAD.WIDE per lane give d - cum * r as 64-bit
//    values whose high words are 0 (cum * r <= d) or -1; their sum is the
//    number of qualifying symbols of the lane (cum is increasing), the ballot
//    of "any" the owner lane;
//  * every lane prepares the (low, range) it would produce if it owned the
//    symbol, so the owner's result is one shuffle away;
//  * the model update is one compare + one predicated add per entry;
//  * the next payload byte is fetched before it is needed.
__device__ __forceinline__ uint32_t sel16x(const uint32_t (&a)[16], uint32_t e, int idx) {
  // a[idx + 1] for idx in [0, 16), with a[16] = e
  uint32_t b[8], c[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) b[i] = (idx & 1) ? (2 * i + 2 < 16 ? a[2 * i + 2] : e) : a[2 * i + 1];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i] = (idx & 2) ? b[2 * i + 1] : b[2 * i];
  const uint32_t d0 = (idx & 4) ? c[1] : c[0], d1 = (idx & 4) ? c[3] : c[2];
  return (idx & 8) ? d1 : d0;
}

// exclusive cumulative counts from per-entry counts (warp scan over lanes)
__device__ __forceinline__ uint32_t cx_build(uint32_t (&cum)[16], uint32_t& end, int lane,
                                             const uint32_t (&cnt)[16]) {
  uint32_t local = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) local += cnt[k];
  uint32_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  uint32_t run = incl - local;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    cum[k] = run;
    run += cnt[k];
  }
  end = run;
  return __shfl_sync(0xffffffffu, incl, 31);          // total
}

__global__ void __launch_bounds__(32)
    k_rc_decode_x(const uint8_t* __restrict__ data, const int64_t* __restrict__ off,
                  const int64_t* __restrict__ len, int64_t n, int16_t* __restrict__ scans,
                  int32_t* __restrict__ status) {
  const int g = blockIdx.x;
  const int lane = threadIdx.x;
  int16_t* scan = scans + (int64_t)g * n;
  {
    const int64_t head = min(n, (int64_t)((16 - ((uintptr_t)scan & 15)) & 15) / 2);
    if (((uintptr_t)scan & 1) == 0) {
      if (lane < head) scan[lane] = 0;
      int4* body = reinterpret_cast<int4*>(scan + head);
      const int64_t nv = (n - head) / 8;
      for (int64_t j = lane; j < nv; j += 32) body[j] = make_int4(0, 0, 0, 0);
      for (int64_t j = head + nv * 8 + lane; j < n; j += 32) scan[j] = 0;
    } else {
      for (int64_t j = lane; j < n; j += 32) scan[j] = 0;
    }
  }
  __syncwarp();
  const uint8_t* src = data + off[g];
  const int64_t nb = len[g];
  int st = 0;
  uint32_t cum[16], end;
  uint32_t total;
  {
    uint32_t cnt[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) cnt[k] = (16 * lane + k) < kAlpha ? 1u : 0u;
    total = cx_build(cum, end, lane, cnt);
  }
  int64_t wbase = 0, p = 0;
  uint32_t w0 = lane < nb ? src[lane] : 0u;
  uint32_t w1 = 32 + lane < nb ? src[32 + lane] : 0u;
  // the byte at p (valid while p < nb), fetched ahead of its use
  auto fetch = [&]() -> uint32_t {
    if (p - wbase >= 32) {
      wbase += 32;
      w0 = w1;
      w1 = wbase + 32 + lane < nb ? src[wbase + 32 + lane] : 0u;
    }
    return __shfl_sync(0xffffffffu, w0, (int)(p - wbase));
  };
  uint32_t state = 0;
  for (int k = 0; k < 4; ++k) {
    if (p >= nb) { st = 1; break; }
    state = (state << 8) | fetch();
    ++p;
  }
  uint32_t bnext = fetch();
  uint32_t low = 0, range = 0xFFFFFFFFu;
  uint32_t t0 = total;                               // lane l: floor(2^32 / (t0 + l))
  uint32_t minv = (uint32_t)(0x100000000ull / (t0 + lane));
  uint32_t mt = __shfl_sync(0xffffffffu, minv, 0);
  int64_t pos = 0, nsym = 0;
  while (st == 0) {
    uint32_t r = __umulhi(range, mt);
    if (range - r * total >= total) ++r;
    // val = min(floor((state - low) / r), total - 1) (rangecoder.py:216-219):
    // compare cum * r against d = min(state - low, total r - 1); state < low
    // (corrupt streams only) clamps like the 64-bit difference
    const uint32_t dd = state < low ? 0xFFFFFFFFu : state - low;
    const uint32_t d32 = min(total * r - 1u, dd);
    const int nr = -(int)r;                          // r < 2^24: total >= 510
    uint32_t b[16];
#pragma unroll
    for (int k = 0; k < 16; ++k)
      b[k] = (uint32_t)((uint64_t)((int64_t)(int)cum[k] * nr + (int64_t)d32) >> 32);
    const uint32_t nle = 16u + sum16(b);
    const unsigned bal = __ballot_sync(0xffffffffu, nle != 0);
    const int owner = 31 - __clz(bal);
    const int kl = nle > 0 ? (int)nle - 1 : 0;
    const uint32_t ca = sel16(cum, kl), cb = sel16x(cum, end, kl);
    const uint32_t cand_low = low + ca * r;          // rangecoder.py:222-223 (carry-less)
    const uint32_t cand_range = (cb - ca) * r;
    low = __shfl_sync(0xffffffffu, cand_low, owner);
    range = __shfl_sync(0xffffffffu, cand_range, owner);
    const int kk = __shfl_sync(0xffffffffu, kl, owner);
    const int sym = owner * 16 + kk;
    // the next symbol's reciprocal, in flight during the renormalisation
    // (replaced below when the batch ends or the model is halved)
    uint32_t mt_n = __shfl_sync(0xffffffffu, minv, (int)((total + 1u - t0) & 31u));
    for (;;) {                                       // rangecoder.py:224-231
      const uint32_t hi = low + range;
      const bool top_differs = hi < low || (low ^ hi) >= (uint32_t)kTop;
      if (top_differs && range >= (uint32_t)kBottom) break;
      if (top_differs) range = (0u - low) & (uint32_t)(kBottom - 1);
      if (p >= nb) { st = 1; break; }
      state = (state << 8) | bnext;
      ++p;
      bnext = fetch();
      low <<= 8;
      range <<= 8;
    }
    if (st) break;
    // model update (rangecoder.py:143-149): symbols above sym gain one
    const int t = lane > owner ? -1 : (lane == owner ? kk : 16);
#pragma unroll
    for (int k = 0; k < 16; ++k)                     // k > t: one compare + one predicated add
      asm("{\n\t.reg .pred p;\n\tsetp.lt.s32 p, %1, %2;\n\t@p add.u32 %0, %0, 1;\n\t}"
          : "+r"(cum[k]) : "r"(t), "r"(k));
    end += (uint32_t)(t - 16) >> 31;
    total += 1;
    if (total >= (uint32_t)kBottom) {
      uint32_t cnt[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t nx = k + 1 < 16 ? cum[k + 1] : end;
        cnt[k] = (nx - cum[k] + 1) / 2;              // 0 stays 0 (s >= 510)
      }
      total = cx_build(cum, end, lane, cnt);
    }
    if (total - t0 >= 32u) {                         // next batch of reciprocals
      t0 = total;
      minv = (uint32_t)(0x100000000ull / (t0 + lane));
      mt_n = __shfl_sync(0xffffffffu, minv, 0);
    }
    mt = mt_n;
    ++nsym;
    if (sym == 0) break;                            // EOS
    if (sym <= 255) {                               // zero run (rangecoder.py:107-110)
      pos += sym;
      if (pos > n) { st = 2; break; }
    } else {
      if (pos >= n) { st = 3; break; }
      if (lane == 0) scan[pos] = (int16_t)(sym <= 382 ? sym - 383 : sym - 382);
      ++pos;
    }
    if (nsym >= (1 << 24)) { st = 4; break; }
  }
  if (lane == 0) status[g] = st;
}

// ---- parallel-model encoder (default) -----------------------------------------
// The ENCODER knows its whole symbol sequence up front, so the adaptive
// model's state before every symbol -- (cum, cnt) of that symbol and the
// running total -- is a function of the sequence prefix, computable in
// parallel; only the range arithmetic itself stays serial.  Five launches:
//   rcp_scan_summary  per 4096-entry scan chunk: first / last non-zero index
//                     and the symbols of every non-zero but the chunk's first
//   rcp_chunk_offsets per stream, over its chunks: the previous non-zero of
//                     each chunk, each chunk's first symbol index, the count
//   rcp_symbolize     per chunk: zero-run + value symbols (rangecoder.py:75-94)
//   rcp_model         per stream: chunks of <= 1024 symbols; per-warp
//                     histograms, their prefix over warps and over the
//                     alphabet, and an in-warp rank give every symbol's
//                     (cum, cnt) = model at chunk start + what precedes it in
//                     the chunk; a chunk ends exactly where the total reaches
//                     2^16 so the halving (rangecoder.py:147-149) falls
//                     between chunks, recorded as a (position, total) event
//   rcp_code          per stream, one warp: the carry-less coder over the
//                     precomputed (cum, cnt) words (rangecoder.py:155-184)
// The scratch layout inside the caller's idx_ws slice of n int64 per stream:
// symbols u16[n+1] | (cum << 16 | cnt) u32[n+1] | chunk records | events.
namespace rcp {
constexpr int kScanChunk = 4096;                  // scan entries per CTA
constexpr int kScanThreads = 256;                 // 16 entries per thread
constexpr int kSymChunk = 1024;                   // symbols per model step
constexpr int kChunkRec = 4;                      // int32 per chunk record

__host__ __device__ __forceinline__ int64_t al16(int64_t x) { return (x + 15) & ~(int64_t)15; }
__host__ __device__ __forceinline__ int64_t n_chunks(int64_t n) {
  return (n + kScanChunk - 1) / kScanChunk;
}
__host__ __device__ __forceinline__ int64_t max_events(int64_t n) { return (n + 1) / 32768 + 4; }
// bytes of scratch one stream needs (checked against the 8 n bytes available)
__host__ __device__ __forceinline__ int64_t ws_bytes(int64_t n) {
  return al16(2 * (n + 1)) + al16(4 * (n + 1)) + al16(4 * kChunkRec * n_chunks(n)) +
         8 * (max_events(n) + 1);
}

struct Ws {
  uint16_t* sym;
  uint32_t* par;
  int32_t* rec;          // per chunk: first, last, internal symbols | prev, offset
  int32_t* ev;           // [0] = symbol count S, [1] = events, then (pos, total) pairs
};

__device__ __forceinline__ Ws ws_of(int64_t* idx_ws, int g, int64_t n) {
  uint8_t* b = reinterpret_cast<uint8_t*>(idx_ws + (int64_t)g * n);
  Ws w;
  w.sym = reinterpret_cast<uint16_t*>(b);
  b += al16(2 * (n + 1));
  w.par = reinterpret_cast<uint32_t*>(b);
  b += al16(4 * (n + 1));
  w.rec = reinterpret_cast<int32_t*>(b);
  b += al16(4 * kChunkRec * n_chunks(n));
  w.ev = reinterpret_cast<int32_t*>(b);
  return w;
}

__device__ __forceinline__ int nrun(int gap) { return (gap + 254) / 255; }   // ceil(gap / 255)

// block-wide exclusive scans over kScanThreads threads (sum / max)
template <bool kMax>
__device__ __forceinline__ int block_excl(int v, int* sh, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc = kMax ? max(inc, t) : inc + t;
  }
  if (lane == 31) sh[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int wv = lane < kScanThreads / 32 ? sh[lane] : (kMax ? -1 : 0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, wv, o);
      if (lane >= o) wv = kMax ? max(wv, t) : wv + t;
    }
    if (lane < kScanThreads / 32) sh[lane] = wv;            // inclusive warp prefixes
  }
  __syncthreads();
  const int before = warp > 0 ? sh[warp - 1] : (kMax ? -1 : 0);
  total = sh[kScanThreads / 32 - 1];
  int ex = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) ex = kMax ? -1 : 0;
  __syncthreads();                                             // sh reusable
  return kMax ? max(before, ex) : before + ex;
}

struct ThreadRun {
  int first, last, internal;
};

__device__ __forceinline__ ThreadRun thread_run(const int16_t* scan, int64_t n, int64_t j0) {
  ThreadRun t{-1, -1, 0};
#pragma unroll 4
  for (int i = 0; i < kScanChunk / kScanThreads; ++i) {
    const int64_t j = j0 + i;
    if (j < n && scan[j] != 0) {
      if (t.first < 0) t.first = (int)j;
      else t.internal += nrun((int)j - t.last - 1) + 1;
      t.last = (int)j;
    }
  }
  return t;
}

__global__ void __launch_bounds__(kScanThreads)
    rcp_scan_summary(const int16_t* __restrict__ scans, int64_t n, int64_t* __restrict__ idx_ws) {
  __shared__ int sh[kScanThreads / 32];
  const int c = blockIdx.x, g = blockIdx.y;
  const int16_t* scan = scans + (int64_t)g * n;
  const int64_t j0 = (int64_t)c * kScanChunk + threadIdx.x * (kScanChunk / kScanThreads);
  const ThreadRun t = thread_run(scan, n, j0);
  int chunk_last;
  const int prev = block_excl<true>(t.last, sh, chunk_last);   // last non-zero of earlier threads
  int gaps = t.internal + (t.first >= 0 && prev >= 0 ? nrun(t.first - prev - 1) + 1 : 0);
  int internal;
  block_excl<false>(gaps, sh, internal);
  // the chunk's first non-zero: the first thread's with one (smallest index)
  int first = t.first >= 0 ? t.first : INT_MAX;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = first;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kScanThreads / 32; ++w) first = min(first, sh[w]);
    int32_t* rec = ws_of(idx_ws, g, n).rec + (int64_t)c * kChunkRec;
    rec[0] = first == INT_MAX ? -1 : first;
    rec[1] = chunk_last;
    rec[2] = internal;
  }
}

// one thread per stream: chunk records -> (previous non-zero, first symbol)
__global__ void rcp_chunk_offsets(int64_t n, int64_t* __restrict__ idx_ws) {
  const int g = blockIdx.x;
  const Ws w = ws_of(idx_ws, g, n);
  const int64_t nc = n_chunks(n);
  int prev = -1, off = 0;
  for (int64_t c = 0; c < nc; ++c) {
    int32_t* rec = w.rec + c * kChunkRec;
    const int first = rec[0], last = rec[1], internal = rec[2];
    rec[0] = prev;                                   // becomes: previous non-zero
    rec[1] = off;                                    //          first symbol index
    if (first >= 0) {
      off += nrun(first - prev - 1) + 1 + internal;
      prev = last;
    }
  }
  w.sym[off] = 0;                                    // EOS
  w.ev[0] = off + 1;                                 // symbols including EOS
}

__global__ void __launch_bounds__(kScanThreads)
    rcp_symbolize(const int16_t* __restrict__ scans, int64_t n, int64_t* __restrict__ idx_ws) {
  __shared__ int sh[kScanThreads / 32];
  const int c = blockIdx.x, g = blockIdx.y;
  const int16_t* scan = scans + (int64_t)g * n;
  const Ws w = ws_of(idx_ws, g, n);
  const int32_t* rec = w.rec + (int64_t)c * kChunkRec;
  const int64_t j0 = (int64_t)c * kScanChunk + threadIdx.x * (kScanChunk / kScanThreads);
  const ThreadRun t = thread_run(scan, n, j0);
  int dummy;
  int prev = block_excl<true>(t.last, sh, dummy);
  prev = max(prev, rec[0]);
  const int nsym = t.first >= 0 ? nrun(t.first - prev - 1) + 1 + t.internal : 0;
  int o = rec[1] + block_excl<false>(nsym, sh, dummy);
  if (t.first < 0) return;
  uint16_t* sym = w.sym;
#pragma unroll 4
  for (int i = 0; i < kScanChunk / kScanThreads; ++i) {
    const int64_t j = j0 + i;
    if (j >= n) break;
    const int v = scan[j];
    if (v == 0) continue;
    int gap = (int)j - prev - 1;                     // rangecoder.py:75-94
    while (gap > 255) {
      sym[o++] = 255;
      gap -= 255;
    }
    if (gap) sym[o++] = (uint16_t)gap;
    sym[o++] = (uint16_t)(v < 0 ? v + 383 : v + 382);
    prev = (int)j;
  }
}

constexpr int kModelThreads = kSymChunk;
constexpr int kAlphaPad = 512;
constexpr int kModelSmem = (32 * kAlphaPad + 3 * kAlphaPad + 32) * 4;

__global__ void __launch_bounds__(kModelThreads, 1)
    rcp_model(int64_t n, int64_t* __restrict__ idx_ws) {
  extern __shared__ uint32_t sm[];
  uint32_t* hist = sm;                               // [32 warps][512]
  uint32_t* cnt = hist + 32 * kAlphaPad;             // model counts at chunk start
  uint32_t* cum = cnt + kAlphaPad;                   // their exclusive prefix
  uint32_t* ccnt = cum + kAlphaPad;                  // this chunk's counts
  uint32_t* red = ccnt + kAlphaPad;                  // 32 scratch words
  const int g = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Ws w = ws_of(idx_ws, g, n);
  const int S = w.ev[0];
  if (tid < kAlphaPad) {
    cnt[tid] = tid < kAlpha ? 1u : 0u;
    cum[tid] = min(tid, kAlpha);
  }
  uint32_t total = kAlpha;
  int nev = 0;
  __syncthreads();
  for (int base = 0; base < S;) {
    const int len = min(min(kSymChunk, S - base), (int)(kBottom - total));
    for (int i = tid; i < 32 * kAlphaPad; i += kModelThreads) hist[i] = 0;
    __syncthreads();
    const bool live = tid < len;
    const int s = live ? w.sym[base + tid] : kAlphaPad - 1;
    if (live) atomicAdd(&hist[warp * kAlphaPad + s], 1u);
    __syncthreads();
    if (tid < kAlphaPad) {                           // exclusive prefix over warps
      uint32_t run = 0;
      for (int ww = 0; ww < 32; ++ww) {
        const uint32_t h = hist[ww * kAlphaPad + tid];
        hist[ww * kAlphaPad + tid] = run;
        run += h;
      }
      ccnt[tid] = run;
    }
    __syncthreads();
    // counts of s in earlier warps, then this warp's row as a prefix over the
    // alphabet: symbols below s in earlier warps
    uint32_t* row = hist + warp * kAlphaPad;
    const uint32_t eq_w = row[s];
    __syncwarp();
    uint32_t loc[16], acc = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      loc[k] = acc;
      acc += row[lane * 16 + k];
    }
    uint32_t inc = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const uint32_t lbase = inc - acc;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k) row[lane * 16 + k] = lbase + loc[k];
    __syncwarp();
    const uint32_t lt_w = row[s];
    uint32_t lt = 0, eq = 0;                         // earlier lanes of this warp
#pragma unroll 8
    for (int j = 0; j < 32; ++j) {
      const int v = __shfl_sync(0xffffffffu, s, j);
      if (j < lane) {
        lt += v < s;
        eq += v == s;
      }
    }
    if (live) w.par[base + tid] = ((cum[s] + lt_w + lt) << 16) | (cnt[s] + eq_w + eq);
    __syncthreads();
    total += (uint32_t)len;
    const bool halve = total >= (uint32_t)kBottom;
    if (tid < kAlphaPad) {
      uint32_t c2 = cnt[tid] + ccnt[tid];
      if (halve) c2 = (c2 + 1) >> 1;                 // rangecoder.py:147-149
      cnt[tid] = c2;
    }
    __syncthreads();
    if (tid < kAlphaPad) {                           // exclusive prefix of cnt
      const uint32_t v = cnt[tid];
      uint32_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += t;
      }
      if (lane == 31) red[warp] = x;
      cum[tid] = x - v;                              // within-warp exclusive
    }
    __syncthreads();
    if (tid < kAlphaPad) {
      uint32_t before = 0;
      for (int ww = 0; ww < warp; ++ww) before += red[ww];
      cum[tid] += before;
    }
    if (halve) {
      uint32_t t2 = 0;
      for (int ww = 0; ww < kAlphaPad / 32; ++ww) t2 += red[ww];
      total = t2;
      if (tid == 0) {
        w.ev[2 + 2 * nev] = base + len;
        w.ev[3 + 2 * nev] = (int32_t)t2;
      }
      ++nev;
    }
    base += len;
    __syncthreads();
  }
  if (tid == 0) w.ev[1] = nev;
}

__global__ void __launch_bounds__(32)
    rcp_code(int64_t n, const int64_t* __restrict__ idx_ws_c, uint8_t* __restrict__ out, int64_t cap,
             int64_t* __restrict__ out_len) {
  const int g = blockIdx.x, lane = threadIdx.x;
  const Ws w = ws_of(const_cast<int64_t*>(idx_ws_c), g, n);
  const int S = w.ev[0], nev = w.ev[1];
  uint8_t* o = out + (int64_t)g * cap;
  int ev = 0;
  int ev_pos = nev > 0 ? w.ev[2] : INT_MAX;
  uint32_t tb = kAlpha;                              // total before symbol `base`
  uint32_t low = 0, range = 0xFFFFFFFFu;
  int64_t pos = 0;
  for (int base = 0; base < S; base += 32) {
    if (base == ev_pos) {                            // the model was halved here
      tb = (uint32_t)w.ev[3 + 2 * ev];
      ++ev;
      ev_pos = ev < nev ? w.ev[2 + 2 * ev] : INT_MAX;
    }
    // per lane, off the serial path: its symbol's (cum, cnt), the total it
    // is coded against (a halving inside the batch restarts the count) and
    // floor(2^32 / total), so the coder's range / total is one multiply-high
    // plus one correction (the estimate is exact or one short)
    const int i = base + lane;
    const uint32_t cc = i < S ? __ldcs(w.par + i) : 0u;
    const bool after = ev_pos < base + 32 && i >= ev_pos;
    const uint32_t ti = after ? (uint32_t)w.ev[3 + 2 * ev] + (uint32_t)(i - ev_pos) : tb + lane;
    const uint32_t mi = (uint32_t)(0x100000000ull / ti);
    const int nb = min(32, S - base);
    uint32_t c_t = __shfl_sync(0xffffffffu, cc, 0), m_t = __shfl_sync(0xffffffffu, mi, 0);
    uint32_t t_t = __shfl_sync(0xffffffffu, ti, 0);
    for (int t = 0; t < nb; ++t) {
      const int tn = t + 1 < 32 ? t + 1 : 31;        // next symbol's words, in flight
      const uint32_t c_n = __shfl_sync(0xffffffffu, cc, tn);
      const uint32_t m_n = __shfl_sync(0xffffffffu, mi, tn);
      const uint32_t t_n = __shfl_sync(0xffffffffu, ti, tn);
      uint32_t r = __umulhi(range, m_t);
      if (range - r * t_t >= t_t) ++r;
      low += (c_t >> 16) * r;                        // < 2^32 + range: carry-less
      range = (c_t & 0xFFFFu) * r;
      // renormalise (rangecoder.py:167-176) on the 33-bit low + range
      while (((uint64_t)low ^ ((uint64_t)low + range)) < kTop || range < kBottom) {
        if (((uint64_t)low ^ ((uint64_t)low + range)) >= kTop) range = (0u - low) & (uint32_t)(kBottom - 1);
        if (lane == 0 && pos < cap) o[pos] = (uint8_t)(low >> 24);
        ++pos;
        low <<= 8;
        range <<= 8;
      }
      c_t = c_n;
      m_t = m_n;
      t_t = t_n;
    }
    if (ev_pos < base + 32 && ev_pos > base) {       // consumed inside this batch
      tb = (uint32_t)w.ev[3 + 2 * ev] + (uint32_t)(base + 32 - ev_pos);
      ++ev;
      ev_pos = ev < nev ? w.ev[2 + 2 * ev] : INT_MAX;
    } else {
      tb += 32;
    }
  }
  for (int k = 0; k < 4; ++k) {                      // rangecoder.py:182-184
    if (lane == 0 && pos < cap) o[pos] = (uint8_t)(low >> 24);
    ++pos;
    low <<= 8;
  }
  if (lane == 0) out_len[g] = pos > cap ? -pos : pos;
}
}  // namespace rcp

// encode_stream for explicit symbol lists (one CTA / thread per stream)
__global__ void k_rc_encode_symbols(const int32_t* __restrict__ syms, const int64_t* __restrict__ off,
                                    const int64_t* __restrict__ len, uint8_t* __restrict__ out,
                                    int64_t cap, int64_t* __restrict__ out_len) {
  __shared__ Model m;
  if (threadIdx.x != 0) return;
  const int g = blockIdx.x;
  for (int s = 0; s < kFen; ++s) m.cnt[s] = s < kAlpha ? 1u : 0u;
  model_build(m);
  Enc e{0, kMask32, out + (int64_t)g * cap, 0, cap, false};
  const int32_t* src = syms + off[g];
  for (int64_t i = 0; i < len[g]; ++i) enc_symbol(e, m, src[i]);
  for (int k = 0; k < 4; ++k) {
    if (e.pos < e.cap) e.out[e.pos] = (uint8_t)((e.low >> 24) & 0xFF);
    else e.overflow = true;
    e.pos += 1;
    e.low = (e.low << 8) & kMask32;
  }
  out_len[g] = e.overflow ? -e.pos : e.pos;
}

// decode_stream to a symbol list (rangecoder.py:188-235); status 1 truncated,
// 4 symbol budget exceeded, 7 output capacity exceeded
__global__ void k_rc_decode_symbols(const uint8_t* __restrict__ src, int64_t nb, int64_t max_symbols,
                                    int64_t cap, int32_t* __restrict__ syms, int64_t* __restrict__ nsym,
                                    int32_t* __restrict__ status) {
  __shared__ Model m;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kFen; ++s) m.cnt[s] = s < kAlpha ? 1u : 0u;
  model_build(m);
  int64_t p = 0, count = 0;
  int st = 0;
  uint64_t state = 0;
  for (int k = 0; k < 4; ++k) {
    if (p >= nb) { st = 1; break; }
    state = (state << 8) | src[p++];
  }
  uint64_t low = 0, range = kMask32;
  while (st == 0) {
    const uint64_t total = m.total;
    const uint64_t r = range / total;
    uint64_t val = (state - low) / r;
    if (val >= total) val = total - 1;
    uint32_t c32;
    const int sym = model_find(m, (uint32_t)val, &c32);
    if (count >= cap) { st = 7; break; }
    syms[count++] = sym;
    const uint64_t c = c32, d = c + m.cnt[sym];
    low += c * r;
    range = (d - c) * r;
    while ((low ^ (low + range)) < kTop || range < kBottom) {
      if ((low ^ (low + range)) >= kTop) range = (kMask32 + 1 - low) & (kBottom - 1);
      if (p >= nb) { st = 1; break; }
      state = ((state << 8) | src[p++]) & kMask32;
      low = (low << 8) & kMask32;
      range <<= 8;
    }
    if (st) break;
    model_update(m, sym);
    if (sym == 0) break;
    if (count >= max_symbols) { st = 4; break; }
  }
  *nsym = count;
  *status = st;
}

}  // namespace sst

using namespace sst;

extern "C" int sst_rc_encode_symbols(const int32_t* syms, const int64_t* off, const int64_t* len,
                                     int G, uint8_t* out, int64_t cap, int64_t* out_len,
                                     void* stream) {
  if (G < 0 || cap < 0) return SST_ERR_ARG;
  if (G == 0) return SST_OK;
  if (!syms || !off || !len || !out || !out_len) return SST_ERR_ARG;
  k_rc_encode_symbols<<<G, 32, 0, static_cast<cudaStream_t>(stream)>>>(syms, off, len, out, cap,
                                                                         out_len);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_rc_decode_symbols(const uint8_t* data, int64_t nbytes, int64_t max_symbols,
                                     int64_t cap, int32_t* syms, int64_t* nsym, int32_t* status,
                                     void* stream) {
  if (nbytes < 0 || cap < 0) return SST_ERR_ARG;
  if (!data || !syms || !nsym || !status) return SST_ERR_ARG;
  k_rc_decode_symbols<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(data, nbytes, max_symbols,
                                                                         cap, syms, nsym, status);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_residual(const float* work, const float* img, int G, int h, int w,
                            double theta, double step, double* avg, int16_t* dense, double* mags,
                            int32_t* count, void* stream) {
  if (G < 0 || h <= 0 || w <= 0 || !(step > 0.0) || theta < 0.0) return SST_ERR_ARG;
  if (G == 0) return SST_OK;
  if (!work || !img || !dense || !count) return SST_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = (int64_t)h * w * 3;
  SST_CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(int32_t) * G, st));
  dim3 grid((unsigned)ceil_div64(n, 256), G);
  k_residual<<<grid, 256, 0, st>>>(work, img, n, theta, step, avg, dense, mags, count);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_mean_axis0(const double* res, int T, int64_t n, double* out, void* stream) {
  if (T < 1 || n < 0) return SST_ERR_ARG;
  if (n == 0) return SST_OK;
  if (!res || !out) return SST_ERR_ARG;
  k_mean_axis0<<<(unsigned)ceil_div64(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      res, T, n, out);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_sparsify(const double* avg, int G, int64_t n, double theta, double step,
                            int16_t* dense, double* mags, int32_t* count, void* stream) {
  if (G < 0 || n < 0 || !(step > 0.0) || theta < 0.0) return SST_ERR_ARG;
  if (G == 0) return SST_OK;
  if (!count || (n > 0 && (!avg || !dense))) return SST_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SST_CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(int32_t) * G, st));
  if (n == 0) return SST_OK;
  dim3 grid((unsigned)ceil_div64(n, 256), G);
  k_sparsify<<<grid, 256, 0, st>>>(avg, n, theta, step, dense, mags, count);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_apply_residual(float* img, const int16_t* dense, const int32_t* count, int G,
                                  int h, int w, double step, void* stream) {
  if (G < 0 || h <= 0 || w <= 0 || !(step > 0.0)) return SST_ERR_ARG;
  if (G == 0) return SST_OK;
  if (!img || !dense || !count) return SST_ERR_ARG;
  const int64_t n = (int64_t)h * w * 3;
  dim3 grid((unsigned)ceil_div64(n, 256), G);
  k_apply_residual<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(img, dense, count, n, step);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_mask_scan(const int16_t* dense, const uint8_t* keep, int64_t total, int16_t* out,
                             void* stream) {
  if (total < 0) return SST_ERR_ARG;
  if (total == 0) return SST_OK;
  if (!dense || !keep || !out) return SST_ERR_ARG;
  k_mask_scan<<<(unsigned)ceil_div64(total, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      dense, keep, total, out);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_rc_encode(const int16_t* scans, int G, int64_t n, int64_t* idx_ws, uint8_t* out,
                             int64_t cap, int64_t* out_len, void* stream) {
  if (G < 0 || n < 0 || cap < 0) return SST_ERR_ARG;
  if (G == 0) return SST_OK;
  if ((n > 0 && (!scans || !idx_ws)) || !out || !out_len) return SST_ERR_ARG;
  // default: the parallel-model encoder (rcp::); A/B: SST_RC=cum (the
  // one-warp cumulative-table coder), SST_RC=fenwick (single thread, Fenwick
  // tree) or SST_RC=warp (warp-reduced counts)
  const char* mode = getenv("SST_RC");
  auto st = static_cast<cudaStream_t>(stream);
  // the parallel-model encoder needs its scratch inside the 8 n bytes per
  // stream and int32 positions; small scans take the one-launch warp coder
  const bool par = n >= rcp::kScanChunk && n < ((int64_t)1 << 30) &&
                   rcp::ws_bytes(n) <= 8 * n && G <= 65535;
  if (mode && mode[0] == 'f') {
    k_rc_encode<<<G, kRcThreads, 0, st>>>(scans, n, idx_ws, out, cap, out_len);
  } else if (mode && mode[0] == 'w') {
    k_rc_encode_w<<<G, kRcThreads, 0, st>>>(scans, n, idx_ws, out, cap, out_len);
  } else if ((mode && mode[0] == 'c') || !par) {
    k_rc_encode_c<<<G, kRcThreadsC, 0, st>>>(scans, n, idx_ws, out, cap, out_len);
  } else {
    static bool attr = false;
    if (!attr) {
      SST_CUDA_TRY(cudaFuncSetAttribute(rcp::rcp_model, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          rcp::kModelSmem));
      attr = true;
    }
    const dim3 chunks((unsigned)rcp::n_chunks(n), G);
    rcp::rcp_scan_summary<<<chunks, rcp::kScanThreads, 0, st>>>(scans, n, idx_ws);
    rcp::rcp_chunk_offsets<<<G, 1, 0, st>>>(n, idx_ws);
    rcp::rcp_symbolize<<<chunks, rcp::kScanThreads, 0, st>>>(scans, n, idx_ws);
    rcp::rcp_model<<<G, rcp::kModelThreads, rcp::kModelSmem, st>>>(n, idx_ws);
    rcp::rcp_code<<<G, 32, 0, st>>>(n, idx_ws, out, cap, out_len);
  }
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_rc_decode(const uint8_t* data, const int64_t* off, const int64_t* len, int G,
                             int64_t n, int16_t* scans, int32_t* status, void* stream) {
  if (G < 0 || n < 0) return SST_ERR_ARG;
  if (G == 0) return SST_OK;
  if (!data || !off || !len || !status || (n > 0 && !scans)) return SST_ERR_ARG;
  const char* mode = getenv("SST_RC");
  auto st = static_cast<cudaStream_t>(stream);
  if (mode && mode[0] == 'f')
    k_rc_decode<<<G, kRcThreads, 0, st>>>(data, off, len, n, scans, status);
  else if (mode && mode[0] == 'w')
    k_rc_decode_w<<<G, kRcThreads, 0, st>>>(data, off, len, n, scans, status);
  else if (mode && mode[0] == 'q')
    k_rc_decode_c<true><<<G, kRcThreadsC, 0, st>>>(data, off, len, n, scans, status);
  else if (mode && mode[0] == 'c')
    k_rc_decode_c<false><<<G, kRcThreadsC, 0, st>>>(data, off, len, n, scans, status);
  else
    k_rc_decode_x<<<G, 32, 0, st>>>(data, off, len, n, scans, status);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

// ---- compat-layer elementwise pieces of residual.py ------------------------
namespace sst {
__global__ void k_residual_diff(const float* __restrict__ x, const float* __restrict__ xh, int64_t n,
                                double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (double)x[i] - (double)xh[i];
}
__global__ void k_dequant_i16(const int16_t* __restrict__ q, int64_t n, double step,
                              double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (double)q[i] * step;
}
}  // namespace sst

// compute_residual (residual.py:62-73): out = float64(x) - float64(x_hat)
extern "C" int sst_residual_diff(const float* x, const float* xh, int64_t n, double* out,
                                 void* stream) {
  if (n < 0) return SST_ERR_ARG;
  if (n == 0) return SST_OK;
  if (!x || !xh || !out) return SST_ERR_ARG;
  k_residual_diff<<<(unsigned)ceil_div64(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      x, xh, n, out);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

// SparseResidual.dense (residual.py:56-59): out = float64(q) * step
extern "C" int sst_dequant_i16(const int16_t* q, int64_t n, double step, double* out, void* stream) {
  if (n < 0) return SST_ERR_ARG;
  if (n == 0) return SST_OK;
  if (!q || !out) return SST_ERR_ARG;
  k_dequant_i16<<<(unsigned)ceil_div64(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      q, n, step, out);
  SST_LAUNCH_CHECK();
  return SST_OK;
}
