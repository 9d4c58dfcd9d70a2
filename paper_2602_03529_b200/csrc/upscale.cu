// K5: reconstruction -- scale_gop(up, crop) + blend_boundary, materialising
// the 9 output frames of each GoP (codec.py:217-296), plus the standalone
// upscale / bilinear / blend / clip-cast / mse entry points.
//
// Bilinear: half-pixel centres, coordinates clipped to [0, n-1], float64 in
// the reference's exact operation order (codec.py:222-235), clip, float32.
// Blend (Eq. 2): alpha*prev + (1-alpha)*curr, alpha = (n-i)/n, float64.
//
// The fused kernel computes each distinct output value once per pixel (I
// upscale, P upscale and -- for boundary frames -- the previous GoP's P
// upscale recomputed from its small working image instead of re-reading two
// full-resolution frames) and streams the 9 frames out.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include <type_traits>

#include "common.cuh"
#include "dct8.cuh"
#include "tma.cuh"

namespace sst {

struct AxisTap {
  int lo, hi;
  double f, g;   // frac, 1 - frac
};

// a row's tap as kept in shared memory: one 16-byte LDS.128 per row (g is
// recomputed as 1 - f, the same double operation axis_tap performs)
struct __align__(16) RowTap {
  int lo, hi;
  double f;
};

// codec.py:222-228
__device__ __forceinline__ AxisTap axis_tap(int o, int n_in, int s) {
  double c = ((double)o + 0.5) / (double)s - 0.5;
  double top = (double)n_in - 1.0;
  c = c < 0.0 ? 0.0 : (c > top ? top : c);
  int lo = (int)floor(c);
  AxisTap t;
  t.lo = lo;
  t.hi = min(lo + 1, n_in - 1);
  t.f = c - (double)lo;
  t.g = 1.0 - t.f;
  return t;
}

__device__ __forceinline__ RowTap to_row(const AxisTap& t) { return RowTap{t.lo, t.hi, t.f}; }
__device__ __forceinline__ AxisTap from_row(const RowTap& r) {
  const uint4 v = *reinterpret_cast<const uint4*>(&r);     // one 16-byte load
  AxisTap t;
  t.lo = (int)v.x;
  t.hi = (int)v.y;
  t.f = __hiloint2double((int)v.w, (int)v.z);
  t.g = 1.0 - t.f;
  return t;
}

// codec.py:233-235: top = a*(1-fx) + b*fx ; bot = ... ; top*(1-fy) + bot*fy
template <typename T>
__device__ __forceinline__ double bilerp(const T* img, int w, const AxisTap& ty, const AxisTap& tx,
                                         int ch) {
  const T* r0 = img + (int64_t)ty.lo * w * 3;
  const T* r1 = img + (int64_t)ty.hi * w * 3;
  double a = (double)r0[tx.lo * 3 + ch], b = (double)r0[tx.hi * 3 + ch];
  double c = (double)r1[tx.lo * 3 + ch], d = (double)r1[tx.hi * 3 + ch];
  double top = a * tx.g + b * tx.f;
  double bot = c * tx.g + d * tx.f;
  return top * ty.g + bot * ty.f;
}

// np.clip(x, 0, 1) for values that are provably >= 0 or -0.0: every K5
// intermediate is a sum of products of non-negative factors (samples in
// [0, 1], bilinear weights f, 1 - f in [0, 1], blend weights in [0, 1]), so
// the lower bound never triggers and -0.0 passes through exactly as in numpy.
__device__ __forceinline__ double clip_hi1(double x) { return x > 1.0 ? 1.0 : x; }

// f32_clip_hi1(x) as one float min: float rounding is monotonic, so
// x > 1 implies (float)x >= 1 and x <= 1 implies (float)x <= 1 -- the result
// is bit-identical (including -0.0) and costs one FMNMX instead of a DSETP and
// two FSELs on the 64-bit value.
__device__ __forceinline__ float f32_clip_hi1(double x) { return fminf((float)x, 1.0f); }

// Blend of boundary frame f (0-based) of a width-kN blend,
// clip(alpha*q + (1-alpha)*u) with alpha = (kN-1-f)/kN (codec.py:289-293), for
// q, u the float32 upscaled samples (in [0, 1], possibly -0.0).  Two weights
// are evaluated in float arithmetic with bit-identical results:
//  * alpha = 0: 0*q + 1*u is exact in either precision; fmaf(0, q, u) keeps
//    IEEE's signed-zero rules (-0 + -0 = -0, -0 + +0 = +0).
//  * alpha = 1/2: 0.5q + 0.5u = (q+u)/2.  When the exponents of q and u are
//    within 28 the float64 sum is exact, so the reference's result is
//    round_f32((q+u)/2); otherwise the smaller addend is < ulp32(larger)/32
//    and both roundings return the larger one / 2.  round_f32((q+u)/2) =
//    round_f32(q+u) * 0.5: binary scaling commutes with rounding while the
//    half is normal, and when q+u < 2^-125 the float sum is exact (both are
//    multiples of 2^-149 below the first binade whose ulp exceeds that) and
//    the float multiply rounds the exact half once.  Signed zeros follow the
//    same IEEE rules in both.  The sum is <= 1: the upper clip is inactive.
// Other weights (n = 3, 4: 2/3, 3/4, ...) stay in float64.
template <int kN, int f>
__device__ __forceinline__ float blend_w(float q, float u, double alpha, double beta) {
  constexpr int num = kN - 1 - f;
  if constexpr (num == 0) {
    return __fmaf_rn(0.0f, q, u);
  } else if constexpr (2 * num == kN) {
    return __fmul_rn(__fadd_rn(q, u), 0.5f);
  } else {
    return f32_clip_hi1(alpha * (double)q + beta * (double)u);
  }
}

// A per-thread copy of a uniform 32-bit value: ptxas keeps it in a vector
// register instead of a uniform one, so `base + f * v` below is ONE
// IMAD.WIDE per address (instead of a uniform-to-vector move plus the
// multiply-add, or a 64-bit add pair, per frame store).
__device__ __forceinline__ int opaque_i32(int v) {
  int r;
  asm volatile("{ .reg .u32 t; mov.u32 t, %%tid.x; and.b32 t, t, 0x80000000; or.b32 %0, %1, t; }"
               : "=r"(r) : "r"(v));
  return r;
}
// element f * fs past p (fs < 2^31, 64-bit product)
template <typename T>
__device__ __forceinline__ T* frame_ptr(T* p, int fs, int f) {
  return reinterpret_cast<T*>(reinterpret_cast<char*>(p) + (int64_t)fs * (int64_t)(sizeof(T) * f));
}

// blend_w with the frame index a run-time value (folded once unrolled)
template <int kN>
__device__ __forceinline__ float blend_rt(int f, float q, float u, double alpha, double beta) {
  const int num = kN - 1 - f;
  if (num == 0) return __fmaf_rn(0.0f, q, u);
  if (2 * num == kN) return __fmul_rn(__fadd_rn(q, u), 0.5f);
  return f32_clip_hi1(alpha * (double)q + beta * (double)u);
}

__device__ __forceinline__ float blend_px(float prev, float curr, double alpha) {
  double v = alpha * (double)prev + (1.0 - alpha) * (double)curr;   // codec.py:293
  return (float)clip01(v);
}

// ---- fused upscale + blend + 9-frame store ----
//
// One thread owns one output float column (pixel x, channel) of a band of
// kUpRows output rows and walks down it.  The bilinear filter is separable in
// the reference's own operation order: top = a*(1-fx) + b*fx is a function of
// (source row, output column) only, so each thread evaluates it once per
// source row and keeps the last two rows in registers; the per-output-row work
// is the vertical mix top*(1-fy) + bot*fy.  The I, P and previous-GoP P images
// are read through L1/L2 (they are 1/s^2 of a frame); the 9 frames are written
// with streaming stores, each warp covering 128 contiguous bytes per frame row.
constexpr int kUpThreads = 128;
constexpr int kUpRows = 32;

struct UpArgs {
  const float* img;            // [G][2][h][w][3]
  int G, h, w, s, H, W;
  const SstPrevDesc* prev;     // [G] or null
  int n;                       // blend width (<= 4 when prev is used)
  double alpha[4], beta[4];    // alpha_i = (n - i) / n, beta = 1 - alpha (i = 1..n)
  float* out;                  // [G][9][H][W][3]
  uint8_t* out8;               // raw-rgb24 output [G][9][H][W][3] (the uint8 entry points)
};

// write_raw_video's quantiser (video.py:143): np.rint(v * 255.0).astype(uint8)
// on float32 samples -- the product rounds to float32 first (a float32 array
// times a Python float stays float32), then rint rounds half to even.  Adding
// 1.5 * 2^23 puts the round-to-nearest-even integer in the low mantissa bits.
__device__ __forceinline__ uint32_t rgb24_q(float v) {
  const float t = __fadd_rn(__fmul_rn(v, 255.0f), 12582912.0f);
  return __float_as_uint(t) & 0xFFu;
}

// store one output sample (float32, or its raw-rgb24 byte)
template <typename TOut>
__device__ __forceinline__ void st_out(TOut* p, float v) {
  if constexpr (sizeof(TOut) == 4) __stcs(p, v);
  else *p = (uint8_t)rgb24_q(v);
}
template <typename TOut>
__device__ __forceinline__ TOut* out_base(const UpArgs& a) {
  if constexpr (sizeof(TOut) == 4) return a.out;
  else return a.out8;
}

struct RowCache {
  int ya, yb;
  double a0, a1, b0, b1;       // horizontal taps of up to two images at rows ya / yb
};

template <int NIMG>
__device__ __forceinline__ void hrow(const float* i0, const float* i1, int w, int y,
                                     const AxisTap& tx, int ch, double* o) {
  const int64_t r = (int64_t)y * w;
  {
    double a = (double)__ldg(i0 + (r + tx.lo) * 3 + ch), b = (double)__ldg(i0 + (r + tx.hi) * 3 + ch);
    o[0] = a * tx.g + b * tx.f;
  }
  if (NIMG == 2) {
    double a = (double)__ldg(i1 + (r + tx.lo) * 3 + ch), b = (double)__ldg(i1 + (r + tx.hi) * 3 + ch);
    o[1] = a * tx.g + b * tx.f;
  }
}

// vertical step for output row taps `ty`; returns the clipped float32 samples
template <int NIMG>
__device__ __forceinline__ void vstep(RowCache& c, const float* i0, const float* i1, int w,
                                      const AxisTap& ty, const AxisTap& tx, int ch, float* u) {
  double lo[2], hi[2];
  if (ty.lo == c.ya) { lo[0] = c.a0; lo[1] = c.a1; }
  else if (ty.lo == c.yb) { lo[0] = c.b0; lo[1] = c.b1; }
  else hrow<NIMG>(i0, i1, w, ty.lo, tx, ch, lo);
  if (ty.hi == ty.lo) { hi[0] = lo[0]; hi[1] = lo[1]; }
  else if (ty.hi == c.ya) { hi[0] = c.a0; hi[1] = c.a1; }
  else if (ty.hi == c.yb) { hi[0] = c.b0; hi[1] = c.b1; }
  else hrow<NIMG>(i0, i1, w, ty.hi, tx, ch, hi);
  c.ya = ty.lo; c.a0 = lo[0]; c.a1 = lo[1];
  c.yb = ty.hi; c.b0 = hi[0]; c.b1 = hi[1];
  u[0] = (float)clip01(lo[0] * ty.g + hi[0] * ty.f);          // codec.py:235
  if (NIMG == 2) u[1] = (float)clip01(lo[1] * ty.g + hi[1] * ty.f);
}

template <typename TOut>
__global__ void __launch_bounds__(kUpThreads) k_upscale_blend(const __grid_constant__ UpArgs a) {
  __shared__ RowTap ty_c[kUpRows], ty_p[kUpRows];
  const int tid = threadIdx.x;
  const int q = blockIdx.x * kUpThreads + tid;       // float column: pixel*3 + channel
  const int oy0 = blockIdx.y * kUpRows;
  const int g = blockIdx.z;
  SstPrevDesc pd;
  pd.p_img = nullptr;
  pd.h = pd.w = pd.s = 1;
  if (a.prev) pd = a.prev[g];
  const bool has_prev = pd.p_img != nullptr;
  if (tid < kUpRows) ty_c[tid] = to_row(axis_tap(oy0 + tid, a.h, a.s));
  else if (has_prev && tid < 2 * kUpRows) ty_p[tid - kUpRows] = to_row(axis_tap(oy0 + tid - kUpRows, pd.h, pd.s));
  __syncthreads();
  if (q >= a.W * 3) return;
  const int ox = q / 3, ch = q - ox * 3;
  const AxisTap tx = axis_tap(ox, a.w, a.s);
  const float* iimg = a.img + (int64_t)g * 2 * a.h * a.w * 3;
  const float* pimg = iimg + (int64_t)a.h * a.w * 3;
  const int64_t fstride = (int64_t)a.H * a.W * 3;
  TOut* o = out_base<TOut>(a) + (int64_t)g * kGop * fstride + (int64_t)oy0 * a.W * 3 + q;
  const int rows = min(kUpRows, a.H - oy0);
  RowCache cc{-1, -1, 0.0, 0.0, 0.0, 0.0};
  if (!has_prev) {
    for (int r = 0; r < rows; ++r, o += a.W * 3) {
      float u[2];
      vstep<2>(cc, iimg, pimg, a.w, from_row(ty_c[r]), tx, ch, u);
      st_out(o, u[0]);
#pragma unroll
      for (int f = 1; f < kGop; ++f) st_out(o + f * fstride, u[1]);
    }
    return;
  }
  const AxisTap txp = axis_tap(ox, pd.w, pd.s);
  RowCache cp{-1, -1, 0.0, 0.0, 0.0, 0.0};
  for (int r = 0; r < rows; ++r, o += a.W * 3) {
    float u[2], uq[2];
    vstep<2>(cc, iimg, pimg, a.w, from_row(ty_c[r]), tx, ch, u);
    vstep<1>(cp, pd.p_img, nullptr, pd.w, from_row(ty_p[r]), txp, ch, uq);
    // frame f < n: alpha*prev[9-n+f] + (1-alpha)*curr[f]  (codec.py:289-293);
    // the previous GoP's tail frames are its unblended P upscale when n <= 4
    st_out(o, (float)clip01(a.alpha[0] * (double)uq[0] + a.beta[0] * (double)u[0]));
#pragma unroll
    for (int f = 1; f < kGop; ++f) {
      float v = u[1];
      if (f < a.n) v = (float)clip01(a.alpha[f] * (double)uq[0] + a.beta[f] * (double)u[1]);
      st_out(o + f * fstride, v);
    }
  }
}

// ---- fused upscale + blend, TMA-store variant (aligned widths) ----
//
// A CTA owns a band of kBand output rows x kTQ output floats of one GoP
// (kTQ threads, one output float column each).
//   setup:  row taps of the band, the band's source windows (I, P, previous
//           P; float32) copied to smem with one batch of coalesced loads;
//   compute: each thread walks its column down the band: the horizontal pass
//           a*(1-fx) + b*fx (codec.py:233) once per source row, cached in
//           registers; the vertical pass top*(1-fy) + bot*fy (codec.py:235)
//           per output row; clip, float32, blend (codec.py:289-293);
//   store:  every kTR rows the n+1 distinct tiles (blended frames 0..n-1, P)
//           leave through one TMA bulk tensor store per output frame (frames
//           n..8 share the P tile); TMA clips the crop edges.
constexpr int kTR = 8;                     // output rows per stored tile
constexpr int kTQ = 256;                   // output floats per tile row (= threads)
constexpr int kWF = (kTQ / 6 + 3) * 3 + 3; // max source floats per window row (s >= 2)
// TMA box rows start on a 16-byte boundary: the window is loaded from
// x = (first column & ~3), up to 3 floats before the first column it needs,
// so the pitch covers kWF + 3 floats.
constexpr int kWF9 = 144;                  // window pitch (floats), 16-byte multiple

template <int BAND>
struct UpTmaSmem {
  static constexpr int kWR = BAND / 2 + 2;   // max source rows per band (s >= 2)
  static constexpr int kWin = (kWR * kWF9 + 31) / 32 * 32;   // floats per window, 128 B aligned
  float win[3][kWin];                      // I, P, previous P windows (row pitch kWF9)
  RowTap ty_c[BAND], ty_p[BAND];
  int wx0[2], wx1[2];                      // window column range (source px) cur / prev
  int xs;                                  // I/P window column shift (TMA alignment)
  uint64_t bar;                            // TMA window loads
};
typedef float UpTile[kTR][kTQ];
template <int BAND>
__host__ __device__ constexpr int tile_off() {
  return (int)((sizeof(UpTmaSmem<BAND>) + 127) / 128 * 128);
}
// dynamic smem: windows + NBUF sets of `ntiles` output tiles (n blended + P)
template <int BAND, int NBUF>
__host__ __device__ constexpr int up_tma_smem(int ntiles) {
  return tile_off<BAND>() + NBUF * ntiles * (int)sizeof(UpTile);
}

__device__ __forceinline__ void load_window(float* win, const float* img, int w, int r0, int r1,
                                           int c0f, int c1f, int tid) {
  const int ncol = c1f - c0f;
  const int lane = tid & 31, wid = tid >> 5;
  for (int j = wid; j <= r1 - r0; j += kTQ / 32) {
    const float* src = img + ((int64_t)(r0 + j) * w) * 3 + c0f;
    float* dst = win + j * kWF9;
#pragma unroll
    for (int c = lane; c < kWF; c += 32)
      if (c < ncol) dst[c] = __ldg(src + c);
  }
}

// cp.async completion for the K5-9 window loads
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// kDirect: the 9 frame values of each output float leave as coalesced
// streaming stores straight from registers (a warp writes 128 contiguous bytes
// of a frame row) instead of smem tiles + TMA bulk stores: no tile barrier,
// no store-read wait, and no tile smem (more CTAs per SM).
template <int kBand, int NBUF, bool kPrev, int kN, bool kDirect = false, bool kTmaIn = false>
__global__ void __launch_bounds__(kTQ)
    k_upscale_blend_tma(const __grid_constant__ CUtensorMap omap, const __grid_constant__ CUtensorMap imap,
                        const __grid_constant__ UpArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  UpTmaSmem<kBand>& S = *reinterpret_cast<UpTmaSmem<kBand>*>(smem_raw);
  UpTile* tiles = reinterpret_cast<UpTile*>(smem_raw + tile_off<kBand>());
  const int tid = threadIdx.x;
  const int q0 = blockIdx.x * kTQ;
  const int oy0 = blockIdx.y * kBand;
  const int g = blockIdx.z;
  SstPrevDesc pd;
  pd.p_img = nullptr;
  pd.h = pd.w = pd.s = 1;
  if (kPrev) pd = a.prev[g];
  const bool has_prev = kPrev && pd.p_img != nullptr;
  const int rows = min(kBand, a.H - oy0);
  const int qlast = min(q0 + kTQ, a.W * 3) - 1;
  if (tid < kBand) S.ty_c[tid] = to_row(axis_tap(oy0 + min(tid, rows - 1), a.h, a.s));
  else if (tid < 2 * kBand) {
    if (has_prev) S.ty_p[tid - kBand] = to_row(axis_tap(oy0 + min(tid - kBand, rows - 1), pd.h, pd.s));
  } else if (tid == 2 * kBand) {
    S.wx0[0] = axis_tap(q0 / 3, a.w, a.s).lo;
    S.wx1[0] = axis_tap(qlast / 3, a.w, a.s).hi;
    S.xs = kTmaIn ? (S.wx0[0] * 3) & 3 : 0;
    if (kTmaIn) {
      mbar_init(&S.bar, 1);
      fence_mbar_init();
    }
  } else if (tid == 2 * kBand + 32 && has_prev) {
    S.wx0[1] = axis_tap(q0 / 3, pd.w, pd.s).lo;
    S.wx1[1] = axis_tap(qlast / 3, pd.w, pd.s).hi;
  }
  __syncthreads();

  const float* iimg = a.img + (int64_t)g * 2 * a.h * a.w * 3;
  const float* pimg = iimg + (int64_t)a.h * a.w * 3;
  const int r0 = S.ty_c[0].lo;
  const int pr0 = has_prev ? S.ty_p[0].lo : 0;
  {
    const int r1 = S.ty_c[rows - 1].hi;
    if (kTmaIn) {
      // I and P windows: one TMA box each from the [G*2][h][w*3] tensor map
      if (tid == 0) {
        constexpr uint32_t kBox = UpTmaSmem<kBand>::kWR * kWF9 * sizeof(float);
        mbar_expect_tx(&S.bar, 2 * kBox);
        tma_load_3d(S.win[0], &imap, S.wx0[0] * 3 - S.xs, r0, 2 * g, &S.bar);
        tma_load_3d(S.win[1], &imap, S.wx0[0] * 3 - S.xs, r0, 2 * g + 1, &S.bar);
      }
    } else {
      load_window(S.win[0], iimg, a.w, r0, r1, S.wx0[0] * 3, S.wx1[0] * 3 + 3, tid);
      load_window(S.win[1], pimg, a.w, r0, r1, S.wx0[0] * 3, S.wx1[0] * 3 + 3, tid);
    }
    if (has_prev)
      load_window(S.win[2], pd.p_img, pd.w, pr0, S.ty_p[rows - 1].hi, S.wx0[1] * 3,
                  S.wx1[1] * 3 + 3, tid);
    if (kTmaIn) mbar_wait(&S.bar, 0);
  }
  __syncthreads();

  const int q = min(q0 + tid, a.W * 3 - 1);       // columns past the crop are clipped by TMA
  const int ox = q / 3, ch = q - ox * 3;
  const int nb = has_prev ? kN : 1;                // tiles 0..nb-1: frames 0..nb-1; tile nb: P
  const AxisTap tx = axis_tap(ox, a.w, a.s);
  const int xl = (tx.lo - S.wx0[0]) * 3 + ch + S.xs, xh = (tx.hi - S.wx0[0]) * 3 + ch + S.xs;
  AxisTap txp = tx;
  int pxl = 0, pxh = 0;
  if (has_prev) {
    txp = axis_tap(ox, pd.w, pd.s);
    pxl = (txp.lo - S.wx0[1]) * 3 + ch;
    pxh = (txp.hi - S.wx0[1]) * 3 + ch;
  }
  int ya = -1, yb = -1, qa = -1, qb = -1;
  double ia = 0, pa = 0, ib = 0, pb = 0, qva = 0, qvb = 0;   // horizontal taps at cached rows
  const int z0 = g * kGop;
  const bool col_ok = q0 + tid < a.W * 3;
  for (int c0 = 0, ci = 0; c0 < rows; c0 += kTR, ++ci) {
    // NBUF tile sets rotate; a set is reused once the TMA store issued NBUF
    // chunks ago has finished reading it
    UpTile* tile = tiles + (ci % NBUF) * (nb + 1);
    if (!kDirect && ci >= NBUF) {
      if (tid == 0) {
        if (NBUF == 1) tma_store_wait_read();
        else tma_store_wait_read_1();
      }
      __syncthreads();
    }
    const int cend = min(c0 + kTR, rows);
    for (int r = c0; r < cend; ++r) {
      const AxisTap ty = from_row(S.ty_c[r]);
      if (ty.lo != ya) {
        if (ty.lo == yb) { ia = ib; pa = pb; }
        else {
          const float* wi = &S.win[0][(ty.lo - r0) * kWF9];
          const float* wp = &S.win[1][(ty.lo - r0) * kWF9];
          ia = (double)wi[xl] * tx.g + (double)wi[xh] * tx.f;
          pa = (double)wp[xl] * tx.g + (double)wp[xh] * tx.f;
        }
        ya = ty.lo;
      }
      if (ty.hi != yb) {
        if (ty.hi == ya) { ib = ia; pb = pa; }
        else {
          const float* wi = &S.win[0][(ty.hi - r0) * kWF9];
          const float* wp = &S.win[1][(ty.hi - r0) * kWF9];
          ib = (double)wi[xl] * tx.g + (double)wi[xh] * tx.f;
          pb = (double)wp[xl] * tx.g + (double)wp[xh] * tx.f;
        }
        yb = ty.hi;
      }
      const float ui = f32_clip_hi1(ia * ty.g + ib * ty.f);
      const float up = f32_clip_hi1(pa * ty.g + pb * ty.f);
      const int rr = r - c0;
      if (kDirect) {
        float fv[kN];
        float f0 = ui;
        if (has_prev) {
          const AxisTap tp = from_row(S.ty_p[r]);
          if (tp.lo != qa) {
            if (tp.lo == qb) qva = qvb;
            else {
              const float* wq = &S.win[2][(tp.lo - pr0) * kWF9];
              qva = (double)wq[pxl] * txp.g + (double)wq[pxh] * txp.f;
            }
            qa = tp.lo;
          }
          if (tp.hi != qb) {
            if (tp.hi == qa) qvb = qva;
            else {
              const float* wq = &S.win[2][(tp.hi - pr0) * kWF9];
              qvb = (double)wq[pxl] * txp.g + (double)wq[pxh] * txp.f;
            }
            qb = tp.hi;
          }
          const double dq = (double)f32_clip_hi1(qva * tp.g + qvb * tp.f);
          f0 = f32_clip_hi1(a.alpha[0] * dq + a.beta[0] * (double)ui);
          const double dp = (double)up;
#pragma unroll
          for (int f = 1; f < kN; ++f) fv[f] = f32_clip_hi1(a.alpha[f] * dq + a.beta[f] * dp);
        }
        if (col_ok) {
          const int64_t fstride = (int64_t)a.H * a.W * 3;
          float* o = a.out + ((int64_t)z0 * a.H + oy0 + r) * (int64_t)a.W * 3 + q0 + tid;
          __stcs(o, f0);
#pragma unroll
          for (int f = 1; f < kGop; ++f)
            __stcs(o + f * fstride, (has_prev && f < kN) ? fv[f] : up);
        }
        continue;
      }
      tile[nb][rr][tid] = up;
      if (has_prev) {
        const AxisTap tp = from_row(S.ty_p[r]);
        if (tp.lo != qa) {
          if (tp.lo == qb) qva = qvb;
          else {
            const float* wq = &S.win[2][(tp.lo - pr0) * kWF9];
            qva = (double)wq[pxl] * txp.g + (double)wq[pxh] * txp.f;
          }
          qa = tp.lo;
        }
        if (tp.hi != qb) {
          if (tp.hi == qa) qvb = qva;
          else {
            const float* wq = &S.win[2][(tp.hi - pr0) * kWF9];
            qvb = (double)wq[pxl] * txp.g + (double)wq[pxh] * txp.f;
          }
          qb = tp.hi;
        }
        const double dq = (double)f32_clip_hi1(qva * tp.g + qvb * tp.f);
        tile[0][rr][tid] = f32_clip_hi1(a.alpha[0] * dq + a.beta[0] * (double)ui);
        const double dp = (double)up;
#pragma unroll
        for (int f = 1; f < kN; ++f) tile[f][rr][tid] = f32_clip_hi1(a.alpha[f] * dq + a.beta[f] * dp);
      } else {
        tile[0][rr][tid] = ui;
      }
    }
    if (kDirect) continue;
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      for (int f = 0; f < kGop; ++f)
        tma_store_3d(&omap, &tile[f < nb ? f : nb][0][0], q0, oy0 + c0, z0 + f);
      tma_store_commit();
    }
  }
  if (!kDirect && tid == 0) tma_store_wait_read();
}

// ---- K5 v2: two output floats per thread, 8-byte streaming stores ----
// The direct-store K5 above issues 9 scalar stores per output float -- ~60 %
// of its ~15 instructions per float (ncu: 823 M warp instructions per 32 GoPs,
// issue-active 63 %).  Here a CTA of 128 threads covers the same 256 output
// floats of a 16-row band, each thread two ADJACENT floats (their own
// horizontal taps; the row taps are shared), and every frame row leaves as
// float2 streaming stores: half the store instructions per float, 256
// contiguous bytes per warp per frame row.  Requires W*3 even (8-byte aligned
// rows) and an 8-byte aligned output; the windows arrive by TMA as before.
constexpr int kV2Threads = kTQ / 2;

template <int kBand, bool kPrev, int kN, typename TOut = float>
__global__ void __launch_bounds__(kV2Threads)
    k_upscale_blend_v2(const __grid_constant__ CUtensorMap imap, const __grid_constant__ UpArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  UpTmaSmem<kBand>& S = *reinterpret_cast<UpTmaSmem<kBand>*>(smem_raw);
  const int tid = threadIdx.x;
  const int q0 = blockIdx.x * kTQ;
  const int oy0 = blockIdx.y * kBand;
  const int g = blockIdx.z;
  SstPrevDesc pd;
  pd.p_img = nullptr;
  pd.h = pd.w = pd.s = 1;
  if (kPrev) pd = a.prev[g];
  const bool has_prev = kPrev && pd.p_img != nullptr;
  const int rows = min(kBand, a.H - oy0);
  const int qlast = min(q0 + kTQ, a.W * 3) - 1;
  if (tid < kBand) S.ty_c[tid] = to_row(axis_tap(oy0 + min(tid, rows - 1), a.h, a.s));
  else if (tid < 2 * kBand) {
    if (has_prev) S.ty_p[tid - kBand] = to_row(axis_tap(oy0 + min(tid - kBand, rows - 1), pd.h, pd.s));
  } else if (tid == 2 * kBand) {
    S.wx0[0] = axis_tap(q0 / 3, a.w, a.s).lo;
    S.wx1[0] = axis_tap(qlast / 3, a.w, a.s).hi;
    S.xs = (S.wx0[0] * 3) & 3;
    mbar_init(&S.bar, 1);
    fence_mbar_init();
  } else if (tid == 2 * kBand + 32 && has_prev) {
    S.wx0[1] = axis_tap(q0 / 3, pd.w, pd.s).lo;
    S.wx1[1] = axis_tap(qlast / 3, pd.w, pd.s).hi;
  }
  __syncthreads();
  const int r0 = S.ty_c[0].lo;
  const int pr0 = has_prev ? S.ty_p[0].lo : 0;
  if (tid == 0) {
    constexpr uint32_t kBox = UpTmaSmem<kBand>::kWR * kWF9 * sizeof(float);
    mbar_expect_tx(&S.bar, 2 * kBox);
    tma_load_3d(S.win[0], &imap, S.wx0[0] * 3 - S.xs, r0, 2 * g, &S.bar);
    tma_load_3d(S.win[1], &imap, S.wx0[0] * 3 - S.xs, r0, 2 * g + 1, &S.bar);
  }
  if (has_prev) {           // load_window with this CTA's 4 warps
    const int pr1 = S.ty_p[rows - 1].hi;
    const int c0f = S.wx0[1] * 3, ncol = S.wx1[1] * 3 + 3 - c0f;
    const int lane = tid & 31, wid = tid >> 5;
    for (int j = wid; j <= pr1 - pr0; j += kV2Threads / 32) {
      const float* src = pd.p_img + ((int64_t)(pr0 + j) * pd.w) * 3 + c0f;
      float* dst = S.win[2] + j * kWF9;
#pragma unroll
      for (int c = lane; c < kWF; c += 32)
        if (c < ncol) dst[c] = __ldg(src + c);
    }
  }
  mbar_wait(&S.bar, 0);
  __syncthreads();

  const int qa0 = q0 + 2 * tid;                    // this thread's two floats
  const bool col_ok = qa0 < a.W * 3;               // W*3 even: qa0 + 1 is in range too
  AxisTap tx[2], txp[2];
  int xl[2], xh[2], pxl[2] = {0, 0}, pxh[2] = {0, 0};
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int q = min(qa0 + u, a.W * 3 - 1);
    const int ox = q / 3, ch = q - ox * 3;
    tx[u] = axis_tap(ox, a.w, a.s);
    xl[u] = (tx[u].lo - S.wx0[0]) * 3 + ch + S.xs;
    xh[u] = (tx[u].hi - S.wx0[0]) * 3 + ch + S.xs;
    txp[u] = tx[u];
    if (has_prev) {
      txp[u] = axis_tap(ox, pd.w, pd.s);
      pxl[u] = (txp[u].lo - S.wx0[1]) * 3 + ch;
      pxh[u] = (txp[u].hi - S.wx0[1]) * 3 + ch;
    }
  }
  int ya = -1, yb = -1, qa = -1, qb = -1;
  double ia[2] = {0, 0}, pa[2] = {0, 0}, ib[2] = {0, 0}, pb[2] = {0, 0};
  double qva[2] = {0, 0}, qvb[2] = {0, 0};
  const int64_t orow = (int64_t)a.W * 3;
  const int fsv = opaque_i32(a.H * a.W * 3);       // frame stride (elements)
  TOut* obase = out_base<TOut>(a) + ((int64_t)g * kGop * a.H + oy0) * orow + qa0;
  for (int r = 0; r < rows; ++r, obase += orow) {
    const AxisTap ty = from_row(S.ty_c[r]);
    if (ty.lo != ya) {
      if (ty.lo == yb) {
#pragma unroll
        for (int u = 0; u < 2; ++u) { ia[u] = ib[u]; pa[u] = pb[u]; }
      } else {
        const float* wi = &S.win[0][(ty.lo - r0) * kWF9];
        const float* wp = &S.win[1][(ty.lo - r0) * kWF9];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          ia[u] = (double)wi[xl[u]] * tx[u].g + (double)wi[xh[u]] * tx[u].f;   // codec.py:233
          pa[u] = (double)wp[xl[u]] * tx[u].g + (double)wp[xh[u]] * tx[u].f;
        }
      }
      ya = ty.lo;
    }
    if (ty.hi != yb) {
      if (ty.hi == ya) {
#pragma unroll
        for (int u = 0; u < 2; ++u) { ib[u] = ia[u]; pb[u] = pa[u]; }
      } else {
        const float* wi = &S.win[0][(ty.hi - r0) * kWF9];
        const float* wp = &S.win[1][(ty.hi - r0) * kWF9];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          ib[u] = (double)wi[xl[u]] * tx[u].g + (double)wi[xh[u]] * tx[u].f;
          pb[u] = (double)wp[xl[u]] * tx[u].g + (double)wp[xh[u]] * tx[u].f;
        }
      }
      yb = ty.hi;
    }
    float ui[2], up[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      ui[u] = f32_clip_hi1(ia[u] * ty.g + ib[u] * ty.f);     // codec.py:235
      up[u] = f32_clip_hi1(pa[u] * ty.g + pb[u] * ty.f);
    }
    float fv[kN][2];
#pragma unroll
    for (int u = 0; u < 2; ++u) fv[0][u] = ui[u];
    if (has_prev) {
      const AxisTap tp = from_row(S.ty_p[r]);
      if (tp.lo != qa) {
        if (tp.lo == qb) {
#pragma unroll
          for (int u = 0; u < 2; ++u) qva[u] = qvb[u];
        } else {
          const float* wq = &S.win[2][(tp.lo - pr0) * kWF9];
#pragma unroll
          for (int u = 0; u < 2; ++u)
            qva[u] = (double)wq[pxl[u]] * txp[u].g + (double)wq[pxh[u]] * txp[u].f;
        }
        qa = tp.lo;
      }
      if (tp.hi != qb) {
        if (tp.hi == qa) {
#pragma unroll
          for (int u = 0; u < 2; ++u) qvb[u] = qva[u];
        } else {
          const float* wq = &S.win[2][(tp.hi - pr0) * kWF9];
#pragma unroll
          for (int u = 0; u < 2; ++u)
            qvb[u] = (double)wq[pxl[u]] * txp[u].g + (double)wq[pxh[u]] * txp[u].f;
        }
        qb = tp.hi;
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {            // codec.py:289-293
        const float qf = f32_clip_hi1(qva[u] * tp.g + qvb[u] * tp.f);
        fv[0][u] = blend_w<kN, 0>(qf, ui[u], a.alpha[0], a.beta[0]);
        if constexpr (kN > 1) fv[kN > 1 ? 1 : 0][u] = blend_w<kN, 1>(qf, up[u], a.alpha[1], a.beta[1]);
        if constexpr (kN > 2) fv[kN > 2 ? 2 : 0][u] = blend_w<kN, 2>(qf, up[u], a.alpha[2], a.beta[2]);
        if constexpr (kN > 3) fv[kN > 3 ? 3 : 0][u] = blend_w<kN, 3>(qf, up[u], a.alpha[3], a.beta[3]);
      }
    }
    if (col_ok) {
      // frame f at obase + f * fsv: one IMAD.WIDE per store address
      if constexpr (sizeof(TOut) == 4) {
        __stcs(reinterpret_cast<float2*>(obase), make_float2(fv[0][0], fv[0][1]));
#pragma unroll
        for (int f = 1; f < kGop; ++f) {
          const float2 v = (has_prev && f < kN) ? make_float2(fv[f < kN ? f : 0][0], fv[f < kN ? f : 0][1])
                                                : make_float2(up[0], up[1]);
          __stcs(reinterpret_cast<float2*>(frame_ptr(obase, fsv, f)), v);
        }
      } else {
        // raw-rgb24: the two samples' bytes as one 16-bit store per frame row
        const unsigned short up8 = (unsigned short)(rgb24_q(up[0]) | (rgb24_q(up[1]) << 8));
        __stcs(reinterpret_cast<unsigned short*>(obase),
               (unsigned short)(rgb24_q(fv[0][0]) | (rgb24_q(fv[0][1]) << 8)));
#pragma unroll
        for (int f = 1; f < kGop; ++f) {
          const unsigned short v =
              (has_prev && f < kN)
                  ? (unsigned short)(rgb24_q(fv[f < kN ? f : 0][0]) | (rgb24_q(fv[f < kN ? f : 0][1]) << 8))
                  : up8;
          __stcs(reinterpret_cast<unsigned short*>(frame_ptr(obase, fsv, f)), v);
        }
      }
    }
  }
}

template <int BAND, typename TOut = float>
static int launch_k5_v2(const CUtensorMap& imap, const UpArgs& a, const SstPrevDesc* prev,
                        int blend_n, cudaStream_t st) {
  dim3 grid(ceil_div(a.W * 3, kTQ), ceil_div(a.H, BAND), a.G);
  if (grid.y > 65535) return SST_ERR_ARG;
  // Residency capped at 4 CTAs/SM by the dynamic smem request (54 KB; the
  // kernel needs 18 KB and 72 registers would allow 7): K5 is bound by its
  // DRAM write stream, and fewer CTAs in flight keep the concurrently written
  // rows of the 9 frames closer together.  Measured in bench.py (64 x 1080p
  // streams, K5 ms per 32-GoP launch): 7/SM 1.248, 5/SM 1.232, 4/SM 1.225,
  // 3/SM 1.255.  SST_K5_SMEM overrides the request (A/B).
  const char* es = getenv("SST_K5_SMEM");
  const int smem = std::max((int)sizeof(UpTmaSmem<BAND>), es ? atoi(es) : 54 * 1024);
  auto kern = k_upscale_blend_v2<BAND, false, 1, TOut>;
  if (prev) {
    switch (blend_n) {
      case 1: kern = k_upscale_blend_v2<BAND, true, 1, TOut>; break;
      case 2: kern = k_upscale_blend_v2<BAND, true, 2, TOut>; break;
      case 3: kern = k_upscale_blend_v2<BAND, true, 3, TOut>; break;
      default: kern = k_upscale_blend_v2<BAND, true, 4, TOut>; break;
    }
  }
  SST_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<grid, kV2Threads, smem, st>>>(imap, a);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

// ---- K5 raw-rgb24: float32 arithmetic, verified against the rint ties ----
// A raw-rgb24 output byte is rint(float32(v * 255)) of the float64-exact
// sample v (video.py:143), so v only has to be known well enough to decide
// which side of a half-integer 255 v falls on.  The whole upscale + blend
// runs in float32 FMA arithmetic (no float64, no XU conversions); a sample
// whose estimate t' = 255 v' lies within tau of a half-integer takes the
// float64 path (the reference's exact operation order, bilinear straight from
// the smem windows) instead.  Bound: with samples in [0, 1] and float32
// weights within 2^-25 of the reference's float64 ones, each bilinear pass
// adds <= 2^-23 (two products, one sum, the weight error) so the upscale is
// within 2^-22 of the real-number value and within 2^-22 + 2^-25 of the
// reference's float32 result; a blend adds <= 5 * 2^-25; so
// |t' - float32(255 v)| <= 255 (2^-22 + 6 * 2^-25) + 2 * 2^-17 = 1.22e-4 <
// tau = 1.25 * 2^-13 = 1.53e-4.  Outside the tau band the two roundings
// agree; inside it the exact path decides (half-integers -- rint's ties --
// included).  The band holds ~0.03 % of samples (tau = 2^-12 before: ~1 %
// more time in the exact path, K5u8 0.716 ms).
constexpr float kU8Tau = 0x1.4p-13f;
constexpr int kK5u8Band = 32;              // output rows per CTA (default; SST_K5U8_BAND)

template <int kBand>
struct UpU8Smem {
  float win[3][UpTmaSmem<kBand>::kWin];    // I, P, previous P windows (row pitch kWF9)
  RowTap ty_c[kBand], ty_p[kBand];
  float2 wy_c[kBand], wy_p[kBand];         // float32 (1 - fy, fy) per row
  uint8_t rc_c[kBand], rc_p[kBand];        // per-row cache actions (as Up9fSmem)
  int wx0[2], wx1[2];
  int xs;
  uint64_t bar;
};

// row-cache action byte of row r of a tap table (bits 0-1: lo -- 1 copy the
// cached hi, 2 load; bits 2-3: hi -- 1 copy the new lo, 2 load)
__device__ __forceinline__ uint8_t row_action(const RowTap* tt, int r) {
  const int plo = r > 0 ? tt[r - 1].lo : -1, phi = r > 0 ? tt[r - 1].hi : -1;
  const int lo = tt[r].lo, hi = tt[r].hi;
  const int al = lo == plo ? 0 : (lo == phi ? 1 : 2);
  const int ah = hi == phi ? 0 : (hi == lo ? 1 : 2);
  return (uint8_t)(al | (ah << 2));
}

// the reference's float32 upscale sample at one window position (codec.py:233-235, clip)
__device__ __forceinline__ float exact_up(const float* win, int r_lo, int r_hi, const AxisTap& ty, int xl,
                                          int xh, const AxisTap& tx) {
  const float* w0 = win + r_lo * kWF9;
  const float* w1 = win + r_hi * kWF9;
  const double top = (double)w0[xl] * tx.g + (double)w0[xh] * tx.f;
  const double bot = (double)w1[xl] * tx.g + (double)w1[xh] * tx.f;
  return f32_clip_hi1(top * ty.g + bot * ty.f);
}

// t = 255 v (the exact product, inside two FMAs) -> its rint byte (bits of
// t + 1.5 * 2^23, where the float32 ulp is 1) and whether t is within tau of
// a tie (d = t - rint(t), one rounding of a value below 1: error <= 2^-25).
// Using the exact product instead of float32(255 v) only removes a rounding
// (2^-17) from the bound above.
__device__ __forceinline__ uint32_t q8_check(float v, bool& near_tie) {
  const float m = __fmaf_rn(v, 255.0f, 12582912.0f);
  const float d = __fmaf_rn(v, 255.0f, -__fsub_rn(m, 12582912.0f));
  near_tie |= fabsf(d) > 0.5f - kU8Tau;
  return __float_as_uint(m) & 0xFFu;
}

// kNC output samples per thread (2: one 16-bit store per frame row; 4: one
// 32-bit store, the row control, tie checks' setup and store addressing
// shared by twice the samples)
template <int kBand, bool kPrev, int kN, int kNC>
__global__ void __launch_bounds__(kTQ / kNC)
    k_upscale_blend_u8f(const __grid_constant__ CUtensorMap imap, const __grid_constant__ UpArgs a) {
  constexpr int kNT = kTQ / kNC;
  constexpr int kWxP = 2 * kBand + (2 * kBand + 32 < kNT ? 32 : 1);   // thread of the previous window's range
  static_assert(kWxP < kNT, "setup threads");
  extern __shared__ __align__(128) uint8_t smem_raw[];
  UpU8Smem<kBand>& S = *reinterpret_cast<UpU8Smem<kBand>*>(smem_raw);
  const int tid = threadIdx.x;
  const int q0 = blockIdx.x * kTQ;
  const int oy0 = blockIdx.y * kBand;
  const int g = blockIdx.z;
  SstPrevDesc pd;
  pd.p_img = nullptr;
  pd.h = pd.w = pd.s = 1;
  if (kPrev) pd = a.prev[g];
  const bool has_prev = kPrev && pd.p_img != nullptr;
  const int rows = min(kBand, a.H - oy0);
  const int qlast = min(q0 + kTQ, a.W * 3) - 1;
  if (tid < kBand) {
    const AxisTap t = axis_tap(oy0 + min(tid, rows - 1), a.h, a.s);
    S.ty_c[tid] = to_row(t);
    S.wy_c[tid] = make_float2((float)t.g, (float)t.f);
  } else if (tid < 2 * kBand) {
    if (has_prev) {
      const AxisTap t = axis_tap(oy0 + min(tid - kBand, rows - 1), pd.h, pd.s);
      S.ty_p[tid - kBand] = to_row(t);
      S.wy_p[tid - kBand] = make_float2((float)t.g, (float)t.f);
    }
  } else if (tid == 2 * kBand) {
    S.wx0[0] = axis_tap(q0 / 3, a.w, a.s).lo;
    S.wx1[0] = axis_tap(qlast / 3, a.w, a.s).hi;
    S.xs = (S.wx0[0] * 3) & 3;
    mbar_init(&S.bar, 1);
    fence_mbar_init();
  } else if (tid == kWxP && has_prev) {
    S.wx0[1] = axis_tap(q0 / 3, pd.w, pd.s).lo;
    S.wx1[1] = axis_tap(qlast / 3, pd.w, pd.s).hi;
  }
  __syncthreads();
  if (tid < kBand) S.rc_c[tid] = row_action(S.ty_c, tid);
  else if (tid < 2 * kBand && has_prev) S.rc_p[tid - kBand] = row_action(S.ty_p, tid - kBand);
  const int r0 = S.ty_c[0].lo;
  const int pr0 = has_prev ? S.ty_p[0].lo : 0;
  if (tid == 0) {
    constexpr uint32_t kBox = UpTmaSmem<kBand>::kWR * kWF9 * sizeof(float);
    mbar_expect_tx(&S.bar, 2 * kBox);
    tma_load_3d(S.win[0], &imap, S.wx0[0] * 3 - S.xs, r0, 2 * g, &S.bar);
    tma_load_3d(S.win[1], &imap, S.wx0[0] * 3 - S.xs, r0, 2 * g + 1, &S.bar);
  }
  if (has_prev) {
    const int pr1 = S.ty_p[rows - 1].hi;
    const int c0f = S.wx0[1] * 3, ncol = S.wx1[1] * 3 + 3 - c0f;
    const int lane = tid & 31, wid = tid >> 5;
    for (int j = wid; j <= pr1 - pr0; j += kNT / 32) {
      const float* src = pd.p_img + ((int64_t)(pr0 + j) * pd.w) * 3 + c0f;
      float* dst = S.win[2] + j * kWF9;
#pragma unroll
      for (int c = lane; c < kWF; c += 32)
        if (c < ncol) dst[c] = __ldg(src + c);
    }
  }
  mbar_wait(&S.bar, 0);
  __syncthreads();

  const int qa0 = q0 + kNC * tid;
  const bool col_ok = qa0 < a.W * 3;
  AxisTap tx[kNC], txp[kNC];
  int xl[kNC], xh[kNC], pxl[kNC], pxh[kNC];
  float gxf[kNC], fxf[kNC], gpf[kNC], fpf[kNC];
#pragma unroll
  for (int u = 0; u < kNC; ++u) {
    pxl[u] = pxh[u] = 0;
    gpf[u] = fpf[u] = 0.f;
    const int q = min(qa0 + u, a.W * 3 - 1);
    const int ox = q / 3, ch = q - ox * 3;
    tx[u] = axis_tap(ox, a.w, a.s);
    xl[u] = (tx[u].lo - S.wx0[0]) * 3 + ch + S.xs;
    xh[u] = (tx[u].hi - S.wx0[0]) * 3 + ch + S.xs;
    gxf[u] = (float)tx[u].g;
    fxf[u] = (float)tx[u].f;
    txp[u] = tx[u];
    if (has_prev) {
      txp[u] = axis_tap(ox, pd.w, pd.s);
      pxl[u] = (txp[u].lo - S.wx0[1]) * 3 + ch;
      pxh[u] = (txp[u].hi - S.wx0[1]) * 3 + ch;
      gpf[u] = (float)txp[u].g;
      fpf[u] = (float)txp[u].f;
    }
  }
  float al[kN], be[kN];
#pragma unroll
  for (int f = 0; f < kN; ++f) {
    al[f] = (float)a.alpha[f];
    be[f] = (float)a.beta[f];
  }
  float ia[kNC], pa[kNC], ib[kNC], pb[kNC], qva[kNC], qvb[kNC];
#pragma unroll
  for (int u = 0; u < kNC; ++u) ia[u] = pa[u] = ib[u] = pb[u] = qva[u] = qvb[u] = 0.f;
  const int64_t orow = (int64_t)a.W * 3;
  const int fsv = opaque_i32(a.H * a.W * 3);
  uint8_t* obase = a.out8 + ((int64_t)g * kGop * a.H + oy0) * orow + qa0;
  for (int r = 0; r < rows; ++r, obase += orow) {
    const RowTap rt = S.ty_c[r];
    const float2 wy = S.wy_c[r];
    const int rc = S.rc_c[r];
    if (rc & 3) {
      if (rc & 1) {
#pragma unroll
        for (int u = 0; u < kNC; ++u) { ia[u] = ib[u]; pa[u] = pb[u]; }
      } else {
        const float* wi = &S.win[0][(rt.lo - r0) * kWF9];
        const float* wp = &S.win[1][(rt.lo - r0) * kWF9];
#pragma unroll
        for (int u = 0; u < kNC; ++u) {
          ia[u] = __fmaf_rn(wi[xl[u]], gxf[u], __fmul_rn(wi[xh[u]], fxf[u]));
          pa[u] = __fmaf_rn(wp[xl[u]], gxf[u], __fmul_rn(wp[xh[u]], fxf[u]));
        }
      }
    }
    if (rc & 12) {
      if (rc & 4) {
#pragma unroll
        for (int u = 0; u < kNC; ++u) { ib[u] = ia[u]; pb[u] = pa[u]; }
      } else {
        const float* wi = &S.win[0][(rt.hi - r0) * kWF9];
        const float* wp = &S.win[1][(rt.hi - r0) * kWF9];
#pragma unroll
        for (int u = 0; u < kNC; ++u) {
          ib[u] = __fmaf_rn(wi[xl[u]], gxf[u], __fmul_rn(wi[xh[u]], fxf[u]));
          pb[u] = __fmaf_rn(wp[xl[u]], gxf[u], __fmul_rn(wp[xh[u]], fxf[u]));
        }
      }
    }
    float ui[kNC], up[kNC];
#pragma unroll
    for (int u = 0; u < kNC; ++u) {
      ui[u] = fminf(__fmaf_rn(ia[u], wy.x, __fmul_rn(ib[u], wy.y)), 1.0f);
      up[u] = fminf(__fmaf_rn(pa[u], wy.x, __fmul_rn(pb[u], wy.y)), 1.0f);
    }
    bool tie[kNC];                                  // per sample column
    uint32_t bf[kN][kNC], bp[kNC];
#pragma unroll
    for (int u = 0; u < kNC; ++u) {
      tie[u] = false;
      bp[u] = q8_check(up[u], tie[u]);
      bf[0][u] = q8_check(ui[u], tie[u]);
    }
    if (has_prev) {
      const RowTap pt = S.ty_p[r];
      const float2 wq = S.wy_p[r];
      const int rp = S.rc_p[r];
      if (rp & 3) {
        if (rp & 1) {
#pragma unroll
          for (int u = 0; u < kNC; ++u) qva[u] = qvb[u];
        } else {
          const float* wv = &S.win[2][(pt.lo - pr0) * kWF9];
#pragma unroll
          for (int u = 0; u < kNC; ++u) qva[u] = __fmaf_rn(wv[pxl[u]], gpf[u], __fmul_rn(wv[pxh[u]], fpf[u]));
        }
      }
      if (rp & 12) {
        if (rp & 4) {
#pragma unroll
          for (int u = 0; u < kNC; ++u) qvb[u] = qva[u];
        } else {
          const float* wv = &S.win[2][(pt.hi - pr0) * kWF9];
#pragma unroll
          for (int u = 0; u < kNC; ++u) qvb[u] = __fmaf_rn(wv[pxl[u]], gpf[u], __fmul_rn(wv[pxh[u]], fpf[u]));
        }
      }
#pragma unroll
      for (int u = 0; u < kNC; ++u) {
        const float qf = fminf(__fmaf_rn(qva[u], wq.x, __fmul_rn(qvb[u], wq.y)), 1.0f);
#pragma unroll
        for (int f = 0; f < kN; ++f)
          bf[f][u] = q8_check(__fmaf_rn(al[f], qf, __fmul_rn(be[f], f == 0 ? ui[u] : up[u])), tie[u]);
      }
    }
    bool any_tie = false;
#pragma unroll
    for (int u = 0; u < kNC; ++u) any_tie |= tie[u];
    if (any_tie) {
      // exact float64 path for the row's samples of the columns near a tie
      // (codec.py:233-235, 289-293)
      const AxisTap ty = from_row(rt);
#pragma unroll
      for (int u = 0; u < kNC; ++u) {
        if (!tie[u]) continue;
        const float eui = exact_up(S.win[0], ty.lo - r0, ty.hi - r0, ty, xl[u], xh[u], tx[u]);
        const float eup = exact_up(S.win[1], ty.lo - r0, ty.hi - r0, ty, xl[u], xh[u], tx[u]);
        bp[u] = rgb24_q(eup);
        bf[0][u] = rgb24_q(eui);
        if (has_prev) {
          const AxisTap tp = from_row(S.ty_p[r]);
          const float eq = exact_up(S.win[2], tp.lo - pr0, tp.hi - pr0, tp, pxl[u], pxh[u], txp[u]);
          bf[0][u] = rgb24_q(blend_w<kN, 0>(eq, eui, a.alpha[0], a.beta[0]));
          if constexpr (kN > 1) bf[kN > 1 ? 1 : 0][u] = rgb24_q(blend_w<kN, 1>(eq, eup, a.alpha[1], a.beta[1]));
          if constexpr (kN > 2) bf[kN > 2 ? 2 : 0][u] = rgb24_q(blend_w<kN, 2>(eq, eup, a.alpha[2], a.beta[2]));
          if constexpr (kN > 3) bf[kN > 3 ? 3 : 0][u] = rgb24_q(blend_w<kN, 3>(eq, eup, a.alpha[3], a.beta[3]));
        }
      }
    }
    if (col_ok) {
      if constexpr (kNC == 2) {
        const unsigned short p8 = (unsigned short)__byte_perm(bp[0], bp[1], 0x0040);
        __stcs(reinterpret_cast<unsigned short*>(obase), (unsigned short)__byte_perm(bf[0][0], bf[0][1], 0x0040));
#pragma unroll
        for (int f = 1; f < kGop; ++f) {
          const unsigned short v = (has_prev && f < kN)
                                       ? (unsigned short)__byte_perm(bf[f < kN ? f : 0][0], bf[f < kN ? f : 0][1], 0x0040)
                                       : p8;
          __stcs(reinterpret_cast<unsigned short*>(frame_ptr(obase, fsv, f)), v);
        }
      } else {
        auto pack4 = [](const uint32_t* v) {
          return __byte_perm(__byte_perm(v[0], v[1], 0x0040), __byte_perm(v[2], v[3], 0x0040), 0x5410);
        };
        const unsigned int p8 = pack4(bp);
        __stcs(reinterpret_cast<unsigned int*>(obase), pack4(bf[0]));
#pragma unroll
        for (int f = 1; f < kGop; ++f) {
          const unsigned int v = (has_prev && f < kN) ? pack4(bf[f < kN ? f : 0]) : p8;
          __stcs(reinterpret_cast<unsigned int*>(frame_ptr(obase, fsv, f)), v);
        }
      }
    }
  }
}

template <int kBand, int kNC>
static int launch_k5_u8f(const CUtensorMap& imap, const UpArgs& a, const SstPrevDesc* prev, int blend_n,
                         cudaStream_t st) {
  dim3 grid(ceil_div(a.W * 3, kTQ), ceil_div(a.H, kBand), a.G);
  if (grid.y > 65535) return SST_ERR_ARG;
  const int smem = (int)sizeof(UpU8Smem<kBand>);
  auto kern = k_upscale_blend_u8f<kBand, false, 1, kNC>;
  if (prev) {
    switch (blend_n) {
      case 1: kern = k_upscale_blend_u8f<kBand, true, 1, kNC>; break;
      case 2: kern = k_upscale_blend_u8f<kBand, true, 2, kNC>; break;
      case 3: kern = k_upscale_blend_u8f<kBand, true, 3, kNC>; break;
      default: kern = k_upscale_blend_u8f<kBand, true, 4, kNC>; break;
    }
  }
  SST_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<grid, kTQ / kNC, smem, st>>>(imap, a);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

// ---- K5 with the decoder fused: working-image windows decoded in smem ----
// k_upscale_blend_v2's body over windows that are not loaded but DECODED
// in place from the dequantised token matrices (sst_unpack_tokens): per
// 16-row band the <= 3 x 7 blocks under the window get decode_gop's
// column IDCT (coefficients (0,0) (1,0) (2,0) in column 0, (0,1) in column
// 1, fct 1/16; the all-zero columns share one result), then the row IDCT of
// exactly the window rows, clip, float32 and the I-concealment of invalid
// P blocks -- K4b's operation sequence (decode.cu k_decode), so the
// windows equal the working images bit for bit.  The previous GoP's P
// window is decoded the same way from its own tokens.  Tokens are 1.5
// bytes per working pixel against 12 for the float32 images: the DRAM
// reads interleaved with K5's 9-frame write stream (which cost ~0.17 ms per
// 32-GoP launch, §5 of DESIGN.md) mostly disappear.  Measured (bench, 64 x
// 1080p streams): 1.49 ms per launch against v2's 1.21 ms (K4 0.13 -> 0.04
// ms): the per-band IDCT prologue (~1300 8-point DCTs per CTA, two
// dependent passes behind barriers) costs more than the reads it saves, so
// StreamBank keeps the unfused path by default (fused=True selects this).
// Overlapping the next band's decode with the current band's stores
// (persistent CTAs) is the open step.
constexpr int kTokBR = 3, kTokBC = 7, kTokNB = kTokBR * kTokBC;   // max blocks under a window

struct UpTokArgs {
  const double* tok;            // [G][2][Ht][Wt][12]
  const uint8_t* pvalid;        // [G][Ht][Wt]
  int G, Ht, Wt, h, w, s, H, W;
  const SstPrevTokDesc* prev;   // [G] or null
  int n;
  double alpha[4], beta[4];
};

struct UpTokSmem {
  float win[3][UpTmaSmem<16>::kWin];      // I, P, previous P windows (row pitch kWF9)
  double tk[2][kTokNB][kChannels];        // tokens of the image pair being decoded
  double s1[2][kTokNB][3][2][8];          // column IDCTs, block columns x = 0, 1
  double zc[8];                           // column IDCT of an all-zero column
  uint8_t valid[kTokNB];
  RowTap ty_c[16], ty_p[16];
  int wx0[2], wx1[2];
};

// decode_gop (codec.py:131-140,160-186) of the window rows r0..r1, columns
// c0..c1 (working pixels) of one GoP's I / concealed-P pair into winI (may
// be null) and winP
__device__ __forceinline__ void k5t_decode_pair(UpTokSmem& S, const double* tok, const uint8_t* pval, int Ht,
                                                int Wt, int r0, int r1, int c0, int c1, float* winI, float* winP,
                                                int tid, int nt) {
  const int br0 = r0 >> 3, bc0 = c0 >> 3;
  const int nbr = (r1 >> 3) - br0 + 1, nbc = (c1 >> 3) - bc0 + 1, nb = nbr * nbc;
  const int64_t img = (int64_t)Ht * Wt * kChannels;
  for (int e = tid; e < 2 * nb * kChannels; e += nt) {
    const int im = e / (nb * kChannels), b = (e / kChannels) % nb, c = e % kChannels;
    const int br = br0 + b / nbc, bc = bc0 + b % nbc;
    S.tk[im][b][c] = tok[im * img + ((int64_t)br * Wt + bc) * kChannels + c];
  }
  for (int b = tid; b < nb; b += nt) S.valid[b] = pval[(int64_t)(br0 + b / nbc) * Wt + bc0 + b % nbc];
  __syncthreads();
  for (int it = tid; it < 2 * nb * 6; it += nt) {          // (image, block, channel, column)
    const int im = it / (nb * 6), b = (it / 6) % nb, ch = (it / 2) % 3, x = it & 1;
    double c[8];
#pragma unroll
    for (int y = 0; y < 8; ++y) c[y] = 0.0;
    const double* v = S.tk[im][b] + ch * 4;
    if (x == 0) { c[0] = v[0]; c[1] = v[2]; c[2] = v[3]; }
    else { c[0] = v[1]; }
    dct3_8<true>(c, 1.0 / 16.0);
#pragma unroll
    for (int y = 0; y < 8; ++y) S.s1[im][b][ch][x][y] = c[y];
  }
  __syncthreads();
  const int nr = r1 - r0 + 1;
  for (int it = tid; it < nr * nbc * 3; it += nt) {        // (window row, block column, channel)
    const int r = it / (nbc * 3), bci = (it / 3) % nbc, ch = it % 3;
    const int R = r0 + r, y = R & 7;
    const int b = ((R >> 3) - br0) * nbc + bci;
    double ci[8], cp[8];
    ci[0] = S.s1[0][b][ch][0][y]; ci[1] = S.s1[0][b][ch][1][y];
    cp[0] = S.s1[1][b][ch][0][y]; cp[1] = S.s1[1][b][ch][1][y];
    const double z = S.zc[y];
#pragma unroll
    for (int x = 2; x < 8; ++x) { ci[x] = z; cp[x] = z; }
    dct3_8<false>(ci, 1.0);
    dct3_8<false>(cp, 1.0);
    const bool keep_p = S.valid[b] != 0;
    const int px0 = (bc0 + bci) * 8;
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      const int px = px0 + x;
      if (px < c0 || px > c1) continue;
      const double iv = clip01(ci[x]);
      const double pv = keep_p ? clip01(cp[x]) : iv;
      const int col = r * kWF9 + (px - c0) * 3 + ch;
      if (winI != nullptr) winI[col] = (float)iv;
      winP[col] = (float)pv;
    }
  }
}

template <bool kPrev, int kN>
__global__ void __launch_bounds__(kV2Threads)
    k_upscale_blend_tok(const __grid_constant__ UpTokArgs t, float* __restrict__ out) {
  constexpr int kBand = 16;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  UpTokSmem& S = *reinterpret_cast<UpTokSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int q0 = blockIdx.x * kTQ;
  const int oy0 = blockIdx.y * kBand;
  const int g = blockIdx.z;
  SstPrevTokDesc pd;
  pd.tok = nullptr;
  pd.pvalid = nullptr;
  pd.h = pd.w = pd.s = pd.Ht = pd.Wt = 1;
  if (kPrev) pd = t.prev[g];
  const bool has_prev = kPrev && pd.tok != nullptr;
  const int rows = min(kBand, t.H - oy0);
  const int qlast = min(q0 + kTQ, t.W * 3) - 1;
  if (tid < kBand) S.ty_c[tid] = to_row(axis_tap(oy0 + min(tid, rows - 1), t.h, t.s));
  else if (tid < 2 * kBand) {
    if (has_prev) S.ty_p[tid - kBand] = to_row(axis_tap(oy0 + min(tid - kBand, rows - 1), pd.h, pd.s));
  } else if (tid == 2 * kBand) {
    S.wx0[0] = axis_tap(q0 / 3, t.w, t.s).lo;
    S.wx1[0] = axis_tap(qlast / 3, t.w, t.s).hi;
    double c[8];
#pragma unroll
    for (int y = 0; y < 8; ++y) c[y] = 0.0;
    dct3_8<true>(c, 1.0 / 16.0);
#pragma unroll
    for (int y = 0; y < 8; ++y) S.zc[y] = c[y];
  } else if (tid == 2 * kBand + 32 && has_prev) {
    S.wx0[1] = axis_tap(q0 / 3, pd.w, pd.s).lo;
    S.wx1[1] = axis_tap(qlast / 3, pd.w, pd.s).hi;
  }
  __syncthreads();
  const int r0 = S.ty_c[0].lo;
  const int pr0 = has_prev ? S.ty_p[0].lo : 0;
  k5t_decode_pair(S, t.tok + (int64_t)g * 2 * t.Ht * t.Wt * kChannels, t.pvalid + (int64_t)g * t.Ht * t.Wt,
                  t.Ht, t.Wt, r0, S.ty_c[rows - 1].hi, S.wx0[0], S.wx1[0], S.win[0], S.win[1], tid, kV2Threads);
  if (has_prev) {
    __syncthreads();                                  // tk / s1 reused
    k5t_decode_pair(S, pd.tok, pd.pvalid, pd.Ht, pd.Wt, pr0, S.ty_p[rows - 1].hi, S.wx0[1], S.wx1[1],
                    nullptr, S.win[2], tid, kV2Threads);
  }
  __syncthreads();

  // ---- k_upscale_blend_v2's body (windows start at column wx0, no shift) ----
  const int qa0 = q0 + 2 * tid;
  const bool col_ok = qa0 < t.W * 3;
  AxisTap tx[2], txp[2];
  int xl[2], xh[2], pxl[2] = {0, 0}, pxh[2] = {0, 0};
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int q = min(qa0 + u, t.W * 3 - 1);
    const int ox = q / 3, ch = q - ox * 3;
    tx[u] = axis_tap(ox, t.w, t.s);
    xl[u] = (tx[u].lo - S.wx0[0]) * 3 + ch;
    xh[u] = (tx[u].hi - S.wx0[0]) * 3 + ch;
    txp[u] = tx[u];
    if (has_prev) {
      txp[u] = axis_tap(ox, pd.w, pd.s);
      pxl[u] = (txp[u].lo - S.wx0[1]) * 3 + ch;
      pxh[u] = (txp[u].hi - S.wx0[1]) * 3 + ch;
    }
  }
  int ya = -1, yb = -1, qa = -1, qb = -1;
  double ia[2] = {0, 0}, pa[2] = {0, 0}, ib[2] = {0, 0}, pb[2] = {0, 0};
  double qva[2] = {0, 0}, qvb[2] = {0, 0};
  const int64_t orow = (int64_t)t.W * 3;
  const int fsv = opaque_i32(t.H * t.W * 3);
  float* obase = out + ((int64_t)g * kGop * t.H + oy0) * orow + qa0;
  for (int r = 0; r < rows; ++r, obase += orow) {
    const AxisTap ty = from_row(S.ty_c[r]);
    if (ty.lo != ya) {
      if (ty.lo == yb) {
#pragma unroll
        for (int u = 0; u < 2; ++u) { ia[u] = ib[u]; pa[u] = pb[u]; }
      } else {
        const float* wi = &S.win[0][(ty.lo - r0) * kWF9];
        const float* wp = &S.win[1][(ty.lo - r0) * kWF9];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          ia[u] = (double)wi[xl[u]] * tx[u].g + (double)wi[xh[u]] * tx[u].f;   // codec.py:233
          pa[u] = (double)wp[xl[u]] * tx[u].g + (double)wp[xh[u]] * tx[u].f;
        }
      }
      ya = ty.lo;
    }
    if (ty.hi != yb) {
      if (ty.hi == ya) {
#pragma unroll
        for (int u = 0; u < 2; ++u) { ib[u] = ia[u]; pb[u] = pa[u]; }
      } else {
        const float* wi = &S.win[0][(ty.hi - r0) * kWF9];
        const float* wp = &S.win[1][(ty.hi - r0) * kWF9];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          ib[u] = (double)wi[xl[u]] * tx[u].g + (double)wi[xh[u]] * tx[u].f;
          pb[u] = (double)wp[xl[u]] * tx[u].g + (double)wp[xh[u]] * tx[u].f;
        }
      }
      yb = ty.hi;
    }
    float ui[2], up[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      ui[u] = f32_clip_hi1(ia[u] * ty.g + ib[u] * ty.f);     // codec.py:235
      up[u] = f32_clip_hi1(pa[u] * ty.g + pb[u] * ty.f);
    }
    float fv[kN][2];
#pragma unroll
    for (int u = 0; u < 2; ++u) fv[0][u] = ui[u];
    if (has_prev) {
      const AxisTap tp = from_row(S.ty_p[r]);
      if (tp.lo != qa) {
        if (tp.lo == qb) {
#pragma unroll
          for (int u = 0; u < 2; ++u) qva[u] = qvb[u];
        } else {
          const float* wq = &S.win[2][(tp.lo - pr0) * kWF9];
#pragma unroll
          for (int u = 0; u < 2; ++u)
            qva[u] = (double)wq[pxl[u]] * txp[u].g + (double)wq[pxh[u]] * txp[u].f;
        }
        qa = tp.lo;
      }
      if (tp.hi != qb) {
        if (tp.hi == qa) {
#pragma unroll
          for (int u = 0; u < 2; ++u) qvb[u] = qva[u];
        } else {
          const float* wq = &S.win[2][(tp.hi - pr0) * kWF9];
#pragma unroll
          for (int u = 0; u < 2; ++u)
            qvb[u] = (double)wq[pxl[u]] * txp[u].g + (double)wq[pxh[u]] * txp[u].f;
        }
        qb = tp.hi;
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {            // codec.py:289-293
        const float qf = f32_clip_hi1(qva[u] * tp.g + qvb[u] * tp.f);
        fv[0][u] = blend_w<kN, 0>(qf, ui[u], t.alpha[0], t.beta[0]);
        if constexpr (kN > 1) fv[kN > 1 ? 1 : 0][u] = blend_w<kN, 1>(qf, up[u], t.alpha[1], t.beta[1]);
        if constexpr (kN > 2) fv[kN > 2 ? 2 : 0][u] = blend_w<kN, 2>(qf, up[u], t.alpha[2], t.beta[2]);
        if constexpr (kN > 3) fv[kN > 3 ? 3 : 0][u] = blend_w<kN, 3>(qf, up[u], t.alpha[3], t.beta[3]);
      }
    }
    if (col_ok) {
      __stcs(reinterpret_cast<float2*>(obase), make_float2(fv[0][0], fv[0][1]));
#pragma unroll
      for (int f = 1; f < kGop; ++f) {
        const float2 v = (has_prev && f < kN) ? make_float2(fv[f < kN ? f : 0][0], fv[f < kN ? f : 0][1])
                                              : make_float2(up[0], up[1]);
        __stcs(reinterpret_cast<float2*>(frame_ptr(obase, fsv, f)), v);
      }
    }
  }
}

// ---- K5-9: all 9 frames per CTA, direct stores ----
// A CTA owns a band of kBand output rows x kTQ output floats of one GoP.  It
// loads the source windows of the GoP's 9 working frames (and of the previous
// GoP's frames 9-n+f for the blended ones) in ONE load phase, then walks its
// column down the band, interpolating the 9 frames per output row with the
// row-cache control shared, and writes each row with coalesced streaming
// stores (a warp covers 128 contiguous bytes of a frame row).
//
// Window loads (kLoad): 0 = register-staged loads, 1 = 4-byte cp.async,
// 2 = one TMA box per frame for the current GoP (3-D tensor map over the
// [G*9][h][w*3] working frames, out-of-range rows / columns zero-filled) with
// cp.async for the previous GoP's windows (their base pointers are per-GoP
// table entries, so they have no single tensor map).
// uint8 windows (the int8 learned tokenizer's q = round(255 x) working
// frames): TMA box rows start on a 16-byte = 16-element boundary, so the
// pitch covers kWF + 15 elements
constexpr int kWF9u8 = 160;
// q/255 table copies: 16 (conflict-free lookups, 32 KB) by default; measured
// with 48-row bands (scripts/k5_9u8_micro.py, 32 x 1080p GoPs, blend n=2):
// s=3 1.361 ms (1 copy, 64 rows: 1.350), s=2 1.637 ms (1 copy: 1.818)
#ifndef SST_K59_LUTC
#define SST_K59_LUTC 16
#endif
constexpr int kLutC = SST_K59_LUTC;
template <typename T>
__host__ __device__ constexpr int k59_pitch() { return sizeof(T) == 1 ? kWF9u8 : kWF9; }

template <int kBand, typename T = float>
struct Up9fGeom {
  static constexpr int kWR = kBand / 2 + 2;                      // max source rows (s >= 2)
  static constexpr int kA = 128 / (int)sizeof(T);                // elements per 128 bytes
  static constexpr int kWin = (kWR * k59_pitch<T>() + kA - 1) / kA * kA;   // elements, 128 B aligned
};

// Window element type T: float (the windows as loaded), or double -- each
// source sample widened ONCE after the load instead of once per use by every
// output column that reads it (the float64 -> float32 -> float64 conversions
// run on the XU pipe, which bounded the float variant at ~61 % XU, 0.75 of
// the HBM roofline).  A double window's loads land, as float32, in the upper
// half of its own slot and are widened in place (read all, sync, write all).
template <int kBand, int kP, typename T = float>
struct Up9fSmem {
  T win[kGop][Up9fGeom<kBand, T>::kWin];
  T winp[kP > 0 ? kP : 1][Up9fGeom<kBand, T>::kWin];   // previous GoP's frames 9-n+f, f < n = kP
  // uint8 windows: sample value of q (= float(q / 255)), kLutC copies
  // interleaved so that lane l reads copy l % kLutC: with 16 copies entry q of
  // copy c sits in bank pair c, and a half-warp's 16 lookups never conflict
  double lut[sizeof(T) == 1 ? 256 * kLutC : 1];
  RowTap ty_c[kBand], ty_p[kBand];
  // per-row actions on the cached horizontal taps (bits 0-1: lo row -- 1 copy
  // the cached hi, 2 load; bits 2-3: hi row -- 1 copy the new lo, 2 load):
  // the row-cache decisions are the same for every thread, made once here
  uint8_t rc_c[kBand], rc_p[kBand];
  int wx0[2], wx1[2];
  int xs;                    // current window's column shift (TMA alignment), 0 for cp.async
  uint64_t bar;
};

// Interpolate frames f0..f0+NF-1 from their windows with the row-cache
// control shared, and stream the rows out; the first NB of them (f0 = 0) are
// blended with the previous GoP's frames 9-n+f.
// landing zone of window w's float32 loads
template <typename T, int kWin>
__device__ __forceinline__ float* k5_9_land(T* w) {
  return reinterpret_cast<float*>(w) + (sizeof(T) == 8 ? kWin : 0);
}

// a window sample as the float64 the reference computes with
template <typename T>
__device__ __forceinline__ double k59_val(const T* w, int i, const double* lut) {
  if constexpr (sizeof(T) == 1) return lut[w[i] * kLutC];   // lut: this lane's copy
  else return (double)w[i];
}

// K5-9, float windows, the alpha = 0 blend frame of a -0.0 current sample:
// 0 * prev + (-0.0) keeps the sign of 0 * prev (codec.py:289-293); prev is
// the previous GoP's frame 8 upscaled at this output sample
__device__ __noinline__ float k59_zero_blend(const UpArgs& a, int g, const RowTap& rt, const AxisTap& txp,
                                             int q) {
  const SstPrevDesc pd = a.prev[g];
  const float* img = pd.p_img + (int64_t)(kGop - 1) * pd.h * pd.w * 3;
  const float qf = f32_clip_hi1(bilerp(img, pd.w, from_row(rt), txp, q % 3));
  return __fmaf_rn(0.0f, qf, -0.0f);
}

template <int kBand, int kP, int NF, int NB, typename T>
__device__ __forceinline__ void k5_9_compute(Up9fSmem<kBand, kP, T>& S, const UpArgs& a, int g,
                                             int f0, int q0, int oy0, int rows,
                                             const AxisTap& tx, int xl, int xh,
                                             const AxisTap& txp, int pxl, int pxh) {
  constexpr bool kU8 = sizeof(T) == 1;
  const int tid = threadIdx.x;
  const double* lutb = S.lut + (kU8 ? (tid & (kLutC - 1)) : 0);
  const int r0 = S.ty_c[0].lo;
  // blended frames f < NB = n: alpha_f = (n - 1 - f) / n; the last one has
  // alpha = 0, i.e. clip(0 * prev + 1 * cur) = cur + 0.0 (exact: prev is
  // finite and >= 0), so only the first n - 1 need the previous GoP
  constexpr int NQ = NB > 0 ? NB - 1 : 0;
  constexpr bool BLEND = NQ > 0;
  const int pr0 = BLEND ? S.ty_p[0].lo : 0;
  const int64_t orow = (int64_t)a.W * 3;
  const int fsv = opaque_i32(a.H * a.W * 3);     // frame stride: one IMAD.WIDE per store
  float* op = a.out + ((int64_t)(g * kGop + f0) * a.H + oy0) * orow + q0 + tid;
  double ia[NF], ib[NF], qva[BLEND ? NQ : 1], qvb[BLEND ? NQ : 1];
#pragma unroll
  for (int j = 0; j < NF; ++j) ia[j] = ib[j] = 0.0;
  for (int r = 0; r < rows; ++r, op += orow) {
    const AxisTap ty = from_row(S.ty_c[r]);
    const int rc = S.rc_c[r];                      // row-cache actions (set up once per CTA)
    if (rc & 3) {
      if (rc & 1) {
#pragma unroll
        for (int j = 0; j < NF; ++j) ia[j] = ib[j];
      } else {
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const T* wr = &S.win[f0 + j][(ty.lo - r0) * k59_pitch<T>()];
          ia[j] = k59_val(wr, xl, lutb) * tx.g + k59_val(wr, xh, lutb) * tx.f;     // codec.py:233
        }
      }
    }
    if (rc & 12) {
      if (rc & 4) {
#pragma unroll
        for (int j = 0; j < NF; ++j) ib[j] = ia[j];
      } else {
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const T* wr = &S.win[f0 + j][(ty.hi - r0) * k59_pitch<T>()];
          ib[j] = k59_val(wr, xl, lutb) * tx.g + k59_val(wr, xh, lutb) * tx.f;
        }
      }
    }
    AxisTap tp = ty;
    if (BLEND) {
      tp = from_row(S.ty_p[r]);
      const int rp = S.rc_p[r];
      if (rp & 3) {
        if (rp & 1) {
#pragma unroll
          for (int j = 0; j < NQ; ++j) qva[j] = qvb[j];
        } else {
#pragma unroll
          for (int j = 0; j < NQ; ++j) {
            const T* wq = &S.winp[j][(tp.lo - pr0) * k59_pitch<T>()];
            qva[j] = k59_val(wq, pxl, lutb) * txp.g + k59_val(wq, pxh, lutb) * txp.f;
          }
        }
      }
      if (rp & 12) {
        if (rp & 4) {
#pragma unroll
          for (int j = 0; j < NQ; ++j) qvb[j] = qva[j];
        } else {
#pragma unroll
          for (int j = 0; j < NQ; ++j) {
            const T* wq = &S.winp[j][(tp.hi - pr0) * k59_pitch<T>()];
            qvb[j] = k59_val(wq, pxl, lutb) * txp.g + k59_val(wq, pxh, lutb) * txp.f;
          }
        }
      }
    }
    if constexpr (kU8) {
      // uint8 windows: every sample is q / 255 in [0, 1] and every weight pair
      // sums to 1 within an ulp, so each result is <= 1 + 2^-50 and its float
      // rounding is <= 1.0f: the upper clip is the identity and is omitted.
      // A row with fy = 0 (every third row at s = 3, the clamped top row) is
      // ia * 1 + ib * 0 = ia exactly (ia >= +0), so it skips the vertical mix.
      if (ty.f == 0.0) {
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const float ui = (float)ia[j];
          float v = ui;
          if (j < NQ) v = blend_rt<NB>(j, (float)(qva[j] * tp.g + qvb[j] * tp.f), ui, a.alpha[j], a.beta[j]);
          __stcs(frame_ptr(op, fsv, j), v);
        }
      } else {
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const float ui = (float)(ia[j] * ty.g + ib[j] * ty.f);   // codec.py:235
          float v = ui;
          if (j < NQ) v = blend_rt<NB>(j, (float)(qva[j] * tp.g + qvb[j] * tp.f), ui, a.alpha[j], a.beta[j]);
          __stcs(frame_ptr(op, fsv, j), v);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const float ui = f32_clip_hi1(ia[j] * ty.g + ib[j] * ty.f);     // codec.py:235
        float v = ui;
        if (j < NQ) {   // codec.py:289-293
          v = blend_rt<NB>(j, f32_clip_hi1(qva[j] * tp.g + qvb[j] * tp.f), ui, a.alpha[j], a.beta[j]);
        } else if (j < NB) {
          // alpha = 0: 0 * prev + cur = cur, except that -0.0 + -0.0 stays
          // -0.0: a -0.0 sample takes the previous GoP's frame 8 from global
          // memory for its sign (its window is not staged)
          v = __float_as_uint(ui) == 0x80000000u ? k59_zero_blend(a, g, S.ty_p[r], txp, q0 + tid) : ui + 0.0f;
        }
        __stcs(frame_ptr(op, fsv, j), v);
      }
    }
  }
}

template <int kLoad>
__device__ __forceinline__ void k5_9_window(float* dst, const float* img, int w, int r0, int r1,
                                            int c0f, int c1f, int tid) {
  const int ncol = c1f - c0f;
  const int lane = tid & 31, wid = tid >> 5;
  for (int j = wid; j <= r1 - r0; j += kTQ / 32) {
    const float* src = img + ((int64_t)(r0 + j) * w) * 3 + c0f;
    float* d = dst + j * kWF9;
#pragma unroll
    for (int c = lane; c < kWF; c += 32) {
      if (c < ncol) {
        if (kLoad == 0)
          d[c] = __ldg(src + c);
        else
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(d + c)),
                       "l"(src + c)
                       : "memory");
      }
    }
  }
}

// byte windows (uint8 working frames), register-staged loads
__device__ __forceinline__ void k5_9_window_u8(uint8_t* dst, const uint8_t* img, int w, int r0, int r1,
                                               int c0f, int c1f, int tid) {
  const int ncol = c1f - c0f;
  const int lane = tid & 31, wid = tid >> 5;
  for (int j = wid; j <= r1 - r0; j += kTQ / 32) {
    const uint8_t* src = img + ((int64_t)(r0 + j) * w) * 3 + c0f;
    uint8_t* d = dst + j * kWF9u8;
#pragma unroll
    for (int c = lane; c < kWF; c += 32)
      if (c < ncol) d[c] = __ldg(src + c);
  }
}

#ifndef SST_K59_U8_MINB
#define SST_K59_U8_MINB 3
#endif
template <int kBand, bool kPrev, int kN, int kLoad, typename T, int kSplit = 5>
__global__ void __launch_bounds__(kTQ, sizeof(T) == 8 ? 2 : (sizeof(T) == 1 ? SST_K59_U8_MINB : 3))
    k_upscale9f(const __grid_constant__ CUtensorMap imap, const __grid_constant__ UpArgs a) {
  constexpr int kP = kPrev ? kN - 1 : 0;      // previous-GoP windows (alpha > 0 frames)
  constexpr int kWin = Up9fGeom<kBand, T>::kWin;
  constexpr bool kU8 = sizeof(T) == 1;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Up9fSmem<kBand, kP, T>& S = *reinterpret_cast<Up9fSmem<kBand, kP, T>*>(smem_raw);
  const int tid = threadIdx.x;
  const int q0 = blockIdx.x * kTQ;
  const int oy0 = blockIdx.y * kBand;
  const int g = blockIdx.z;
  SstPrevDesc pd;
  pd.p_img = nullptr;
  pd.h = pd.w = pd.s = 1;
  if (kPrev) pd = a.prev[g];
  const bool has_prev = kPrev && pd.p_img != nullptr;
  const int rows = min(kBand, a.H - oy0);
  const int qlast = min(q0 + kTQ, a.W * 3) - 1;
  if (tid < kBand) S.ty_c[tid] = to_row(axis_tap(oy0 + min(tid, rows - 1), a.h, a.s));
  else if (tid < 2 * kBand) {
    if (has_prev) S.ty_p[tid - kBand] = to_row(axis_tap(oy0 + min(tid - kBand, rows - 1), pd.h, pd.s));
  } else if (tid == 2 * kBand) {
    S.wx0[0] = axis_tap(q0 / 3, a.w, a.s).lo;
    S.wx1[0] = axis_tap(qlast / 3, a.w, a.s).hi;
    S.xs = kLoad == 2 ? (S.wx0[0] * 3) & (kU8 ? 15 : 3) : 0;
    if (kLoad == 2) {
      mbar_init(&S.bar, 1);
      fence_mbar_init();
    }
  } else if (tid == 2 * kBand + 32 && has_prev) {
    S.wx0[1] = axis_tap(q0 / 3, pd.w, pd.s).lo;
    S.wx1[1] = axis_tap(qlast / 3, pd.w, pd.s).hi;
  }
  if (kU8) {                                   // kTQ = 256 threads; consecutive stores
#pragma unroll
    for (int k = 0; k < kLutC; ++k) {
      const int e = k * kTQ + tid;
      // float32(q) / 255 exactly, division-free: q * 0x01010100 + 2^(msb(q)+1)
      // = f(q) * 2^32 (encode.cu, k_encode_u8; all 256 values checked)
      const uint32_t q = (uint32_t)(e / kLutC);
      const uint64_t n = (uint64_t)q * 0x01010100u + (q ? 2u << (31 - __clz(q)) : 0u);
      S.lut[e] = __dmul_rn(__dadd_rn(__hiloint2double((int)((uint32_t)(n >> 32) | 0x43300000u),
                                                      (int)(uint32_t)n), -4503599627370496.0), 0x1p-32);
    }
  }
  __syncthreads();
  if (tid < kBand) S.rc_c[tid] = row_action(S.ty_c, tid);
  else if (tid < 2 * kBand && has_prev) S.rc_p[tid - kBand] = row_action(S.ty_p, tid - kBand);

  // ---- load phase ----
  {
    const int r0 = S.ty_c[0].lo, r1 = S.ty_c[rows - 1].hi;
    if (kLoad == 2) {
      if (tid == 0) {
        constexpr uint32_t kBox =
            Up9fGeom<kBand, T>::kWR * k59_pitch<T>() * (kU8 ? 1 : (uint32_t)sizeof(float));
        mbar_expect_tx(&S.bar, kGop * kBox);
#pragma unroll 1
        for (int f = 0; f < kGop; ++f) {
          void* dst = kU8 ? (void*)S.win[f] : (void*)k5_9_land<T, kWin>(S.win[f]);
          tma_load_3d(dst, &imap, S.wx0[0] * 3 - S.xs, r0, g * kGop + f, &S.bar);
        }
      }
    } else if constexpr (kU8) {
      const int64_t fimg = (int64_t)a.h * a.w * 3;
      const uint8_t* cur = reinterpret_cast<const uint8_t*>(a.img) + (int64_t)g * kGop * fimg;
#pragma unroll 1
      for (int f = 0; f < kGop; ++f)
        k5_9_window_u8(S.win[f], cur + f * fimg, a.w, r0, r1, S.wx0[0] * 3, S.wx1[0] * 3 + 3, tid);
    } else {
      const int64_t fimg = (int64_t)a.h * a.w * 3;
      const float* cur = a.img + (int64_t)g * kGop * fimg;
#pragma unroll 1
      for (int f = 0; f < kGop; ++f)
        k5_9_window<kLoad>(k5_9_land<T, kWin>(S.win[f]), cur + f * fimg, a.w, r0, r1,
                           S.wx0[0] * 3, S.wx1[0] * 3 + 3, tid);
    }
    if (has_prev) {
      const int pr0 = S.ty_p[0].lo, pr1 = S.ty_p[rows - 1].hi;
      const int64_t pimg = (int64_t)pd.h * pd.w * 3;
#pragma unroll
      for (int j = 0; j < kP; ++j) {
        if constexpr (kU8)
          k5_9_window_u8(S.winp[j], reinterpret_cast<const uint8_t*>(pd.p_img) + (kGop - kN + j) * pimg,
                         pd.w, pr0, pr1, S.wx0[1] * 3, S.wx1[1] * 3 + 3, tid);
        else
          k5_9_window<kLoad == 0 ? 0 : 1>(k5_9_land<T, kWin>(S.winp[j]), pd.p_img + (kGop - kN + j) * pimg,
                                          pd.w, pr0, pr1, S.wx0[1] * 3, S.wx1[1] * 3 + 3, tid);
      }
    }
    if (kLoad != 0) cp_async_wait_all();
    if (kLoad == 2) mbar_wait(&S.bar, 0);
    __syncthreads();
    if constexpr (sizeof(T) == 8) {
      // widen every window in place: each thread reads its samples of one
      // window into registers, then (after the barrier) writes them back as
      // doubles over the float32 landing zone
      constexpr int n = Up9fGeom<kBand>::kWR * kWF9;
      constexpr int per = (n + kTQ - 1) / kTQ;
      const int nw = kGop + (has_prev ? kP : 0);
#pragma unroll 1
      for (int f = 0; f < nw; ++f) {
        T* wd = f < kGop ? S.win[f] : S.winp[f - kGop];
        const float* src = k5_9_land<T, kWin>(wd);
        float v[per];
#pragma unroll
        for (int k = 0; k < per; ++k) {
          const int i = tid + k * kTQ;
          v[k] = i < n ? src[i] : 0.0f;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < per; ++k) {
          const int i = tid + k * kTQ;
          if (i < n) wd[i] = (double)v[k];
        }
        __syncthreads();
      }
    }
  }

  if (q0 + tid >= a.W * 3) return;
  const int q = q0 + tid;
  const int ox = q / 3, ch = q - ox * 3;
  const AxisTap tx = axis_tap(ox, a.w, a.s);
  const int xl = (tx.lo - S.wx0[0]) * 3 + ch + S.xs, xh = (tx.hi - S.wx0[0]) * 3 + ch + S.xs;
  if (has_prev) {
    const AxisTap txp = axis_tap(ox, pd.w, pd.s);
    const int pxl = (txp.lo - S.wx0[1]) * 3 + ch, pxh = (txp.hi - S.wx0[1]) * 3 + ch;
    // frames 0..4 (the n <= 4 blended ones first), then 5..8.  Measured
    // slower (32 x 1080p GoPs, s=3, n=2; 1.77 ms here): one 9-frame pass at
    // 3 CTAs/SM 2.07 ms (spills), at 2 CTAs/SM 1.93 ms; this split at 2
    // CTAs/SM 2.10 ms; a 2 + 7 split 1.79 ms
    if constexpr (kSplit >= kGop) {
      k5_9_compute<kBand, kP, kGop, kN>(S, a, g, 0, q0, oy0, rows, tx, xl, xh, txp, pxl, pxh);
    } else {
      k5_9_compute<kBand, kP, kSplit, kN>(S, a, g, 0, q0, oy0, rows, tx, xl, xh, txp, pxl, pxh);
      k5_9_compute<kBand, kP, kGop - kSplit, 0>(S, a, g, kSplit, q0, oy0, rows, tx, xl, xh, txp, pxl, pxh);
    }
  } else {
    k5_9_compute<kBand, kP, kGop, 0>(S, a, g, 0, q0, oy0, rows, tx, xl, xh, tx, 0, 0);
  }
}

template <int BAND, int LOAD, typename T, int SPLIT = 5>
static int launch_k5_9f(const CUtensorMap& imap, const UpArgs& a, const SstPrevDesc* prev,
                        int blend_n, cudaStream_t st) {
  dim3 grid(ceil_div(a.W * 3, kTQ), ceil_div(a.H, BAND), a.G);
  if (grid.y > 65535) return SST_ERR_ARG;
  int smem = (int)sizeof(Up9fSmem<BAND, 0, T>);
  auto kern = k_upscale9f<BAND, false, 1, LOAD, T, SPLIT>;
  if (prev) {
    switch (blend_n) {
      case 1: kern = k_upscale9f<BAND, true, 1, LOAD, T, SPLIT>; smem = sizeof(Up9fSmem<BAND, 0, T>); break;
      case 2: kern = k_upscale9f<BAND, true, 2, LOAD, T, SPLIT>; smem = sizeof(Up9fSmem<BAND, 1, T>); break;
      case 3: kern = k_upscale9f<BAND, true, 3, LOAD, T, SPLIT>; smem = sizeof(Up9fSmem<BAND, 2, T>); break;
      default: kern = k_upscale9f<BAND, true, 4, LOAD, T, SPLIT>; smem = sizeof(Up9fSmem<BAND, 3, T>); break;
    }
  }
  if (const char* es = getenv("SST_K59_SMEM")) smem = std::max(smem, atoi(es));   // A/B: cap CTAs/SM
  SST_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<grid, kTQ, smem, st>>>(imap, a);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

// ---- standalone kernels ----
template <typename Tin, typename Tout, bool kClip>
__global__ void k_upscale(const Tin* __restrict__ img, int64_t n, int h, int w, int s, int ch_out,
                          int cw_out, Tout* __restrict__ out) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = n * ch_out * cw_out * 3;
  if (e >= total) return;
  int ch = (int)(e % 3);
  int64_t t = e / 3;
  int x = (int)(t % cw_out);
  t /= cw_out;
  int y = (int)(t % ch_out);
  int64_t f = t / ch_out;
  AxisTap ay = axis_tap(y, h, s), ax = axis_tap(x, w, s);
  double v = bilerp(img + f * h * w * 3, w, ay, ax, ch);
  if (kClip) v = clip01(v);
  out[e] = (Tout)v;
}

__global__ void k_clip_cast(const double* __restrict__ x, int64_t n, float* __restrict__ out) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) out[e] = (float)clip01(x[e]);
}

__global__ void k_blend(const float* __restrict__ prev, const float* curr, int G, int64_t fe, int n,
                        float* out) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)G * fe) return;
  int64_t g = e / fe, q = e % fe;
  const float* pg = prev + g * kGop * fe;
  const float* cg = curr + g * kGop * fe;
  float* og = out + g * kGop * fe;
  for (int i = 1; i <= n; ++i) {
    double alpha = (double)(n - i) / (double)n;
    og[(i - 1) * fe + q] = blend_px(pg[(kGop - n + i - 1) * fe + q], cg[(i - 1) * fe + q], alpha);
  }
  if (og != cg)
    for (int f = n; f < kGop; ++f) og[f * fe + q] = cg[f * fe + q];
}

}  // namespace sst

using namespace sst;

template <int BAND, int NBUF, bool DIRECT = false, bool TMAIN = false>
static int launch_k5(const CUtensorMap& omap, const CUtensorMap& imap, const UpArgs& a,
                     const SstPrevDesc* prev, int blend_n, cudaStream_t st) {
  dim3 grid(ceil_div(a.W * 3, kTQ), ceil_div(a.H, BAND), a.G);
  if (grid.y > 65535) return SST_ERR_ARG;
  const int smem = DIRECT ? tile_off<BAND>() : up_tma_smem<BAND, NBUF>((prev ? blend_n : 1) + 1);
  auto kern = k_upscale_blend_tma<BAND, NBUF, false, 1, DIRECT, TMAIN>;
  if (prev) {
    switch (blend_n) {
      case 1: kern = k_upscale_blend_tma<BAND, NBUF, true, 1, DIRECT, TMAIN>; break;
      case 2: kern = k_upscale_blend_tma<BAND, NBUF, true, 2, DIRECT, TMAIN>; break;
      case 3: kern = k_upscale_blend_tma<BAND, NBUF, true, 3, DIRECT, TMAIN>; break;
      default: kern = k_upscale_blend_tma<BAND, NBUF, true, 4, DIRECT, TMAIN>; break;
    }
  }
  SST_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<grid, kTQ, smem, st>>>(omap, imap, a);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_upscale_blend(const float* img, int G, int h, int w, int s, int H, int W,
                                 const SstPrevDesc* prev, int blend_n, float* out, void* stream) {
  if (G < 0 || h <= 0 || w <= 0 || H <= 0 || W <= 0) return SST_ERR_ARG;
  if (s != 2 && s != 3) return SST_ERR_ARG;
  if (H > h * s || W > w * s) return SST_ERR_ARG;
  if (blend_n < 1 || blend_n > 8) return SST_ERR_ARG;
  if (prev && blend_n > 4) return SST_ERR_UNSUPPORTED;
  if (G == 0) return SST_OK;
  if (!img || !out) return SST_ERR_ARG;
  if (G > 65535) return SST_ERR_ARG;
  UpArgs a{};
  a.img = img; a.G = G; a.h = h; a.w = w; a.s = s; a.H = H; a.W = W;
  a.prev = prev; a.n = blend_n; a.out = out;
  for (int i = 1; i <= 4; ++i) {
    a.alpha[i - 1] = (double)(blend_n - i) / (double)blend_n;   // python (n - i) / n
    a.beta[i - 1] = 1.0 - a.alpha[i - 1];
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUtensorMap omap;
  memset(&omap, 0, sizeof(omap));
  const char* var = getenv("SST_K5_VARIANT");          // A/B switch for profiling
  const bool want_tma = !(var && var[0] == '2');
  if (want_tma &&
      make_tmap_f32_3d(&omap, out, (uint64_t)W * 3, (uint64_t)H, (uint64_t)G * kGop, kTQ, kTR)) {
    // Default: 16-row bands, one tile set.  Measured in bench.py (64 x 1080p
    // streams): band 16 / 1 set 1.24 ms per 32-GoP launch (0.94 of the HBM
    // peak), band 32 / 1 set 1.27 ms, band 32 / 2 sets 1.54 ms -- the second
    // tile set costs occupancy (the blend variant holds n+1 tiles per set).
    const char* eb = getenv("SST_K5_BAND");       // A/B switches for profiling
    const char* en = getenv("SST_K5_NBUF");
    const int band = (eb && atoi(eb) == 32) ? 32 : 16;
    const int nbuf = (en && atoi(en) == 2) ? 2 : 1;
    // I/P windows by TMA when img admits a tensor map ([G*2][h][w*3]; the
    // register-staged loads otherwise, or with SST_K5_LOAD=sync).  Same time
    // either way (1.17 ms per 32-GoP launch, scripts/k5_ab.sh): K5 is bound
    // by its 7.2 GB of writes, the load phase is hidden by the other CTAs.
    const char* el = getenv("SST_K5_LOAD");
    CUtensorMap imap;
    memset(&imap, 0, sizeof(imap));
    const bool tma_in = band == 16 && nbuf == 1 && !(el && !strcmp(el, "sync")) &&
                        make_tmap_f32_3d(&imap, img, (uint64_t)w * 3, (uint64_t)h,
                                         (uint64_t)G * 2, kWF9, UpTmaSmem<16>::kWR);
    // Default: the direct-store variant with TMA window loads (s=3 with
    // blend: 1.13 ms per 32-GoP launch vs 1.17 ms for TMA-store tiles; a
    // write-only kernel with the same band pattern and no compute reaches
    // 1.03 ms, scripts/diag/write_pattern.py).  SST_K5_VARIANT=tiles: the
    // TMA-store tile variant.
    if (!(var && !strcmp(var, "tiles"))) {        // "direct": streaming stores, no TMA tiles
      // v2 (default when rows and output are 8-byte aligned): two floats per
      // thread, float2 stores; SST_K5_VARIANT=v1: one float per thread
      const bool v2 = tma_in && !(var && !strcmp(var, "v1")) && (W * 3) % 2 == 0 &&
                      (reinterpret_cast<uintptr_t>(out) & 7u) == 0;
      if (v2) return launch_k5_v2<16>(imap, a, prev, blend_n, st);
      if (tma_in) return launch_k5<16, 1, true, true>(omap, imap, a, prev, blend_n, st);
      return band == 16 ? launch_k5<16, 1, true>(omap, omap, a, prev, blend_n, st)
                        : launch_k5<32, 1, true>(omap, omap, a, prev, blend_n, st);
    }
    if (tma_in) return launch_k5<16, 1, false, true>(omap, imap, a, prev, blend_n, st);
    return band == 16 ? (nbuf == 1 ? launch_k5<16, 1>(omap, imap, a, prev, blend_n, st)
                                   : launch_k5<16, 2>(omap, imap, a, prev, blend_n, st))
                      : (nbuf == 1 ? launch_k5<32, 1>(omap, imap, a, prev, blend_n, st)
                                   : launch_k5<32, 2>(omap, imap, a, prev, blend_n, st));
  }
  dim3 grid(ceil_div(W * 3, kUpThreads), ceil_div(H, kUpRows), G);
  if (grid.y > 65535) return SST_ERR_ARG;
  k_upscale_blend<float><<<grid, kUpThreads, 0, st>>>(a);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_upscale_blend_tok(const double* tok, const uint8_t* pvalid, int G, int Ht, int Wt,
                                     int h, int w, int s, int H, int W, const SstPrevTokDesc* prev,
                                     int blend_n, float* out, void* stream) {
  if (G < 0 || h <= 0 || w <= 0 || H <= 0 || W <= 0) return SST_ERR_ARG;
  if (s != 2 && s != 3) return SST_ERR_ARG;
  if (H > h * s || W > w * s) return SST_ERR_ARG;
  if (Ht != ceil_div(h, kBlock) || Wt != ceil_div(w, kBlock)) return SST_ERR_ARG;
  if (blend_n < 1 || blend_n > 8) return SST_ERR_ARG;
  if (prev && blend_n > 4) return SST_ERR_UNSUPPORTED;
  if (G == 0) return SST_OK;
  if (!tok || !pvalid || !out) return SST_ERR_ARG;
  if (G > 65535) return SST_ERR_ARG;
  if ((W * 3) % 2 != 0 || (reinterpret_cast<uintptr_t>(out) & 7u) != 0) return SST_ERR_UNSUPPORTED;
  UpTokArgs t{};
  t.tok = tok; t.pvalid = pvalid;
  t.G = G; t.Ht = Ht; t.Wt = Wt; t.h = h; t.w = w; t.s = s; t.H = H; t.W = W;
  t.prev = prev; t.n = blend_n;
  for (int i = 1; i <= 4; ++i) {
    t.alpha[i - 1] = (double)(blend_n - i) / (double)blend_n;
    t.beta[i - 1] = 1.0 - t.alpha[i - 1];
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  dim3 grid(ceil_div(W * 3, kTQ), ceil_div(H, 16), G);
  if (grid.y > 65535) return SST_ERR_ARG;
  // no residency cap: the per-band decode prologue wants CTAs in flight
  // (measured 1.49 ms per 32-GoP launch uncapped, 1.66 ms at v2's 4 CTAs/SM);
  // SST_K5T_SMEM raises the dynamic-smem request (A/B)
  const char* es = getenv("SST_K5T_SMEM");
  const int smem = std::max((int)sizeof(UpTokSmem), es ? atoi(es) : 0);
  auto kern = k_upscale_blend_tok<false, 1>;
  if (prev) {
    switch (blend_n) {
      case 1: kern = k_upscale_blend_tok<true, 1>; break;
      case 2: kern = k_upscale_blend_tok<true, 2>; break;
      case 3: kern = k_upscale_blend_tok<true, 3>; break;
      default: kern = k_upscale_blend_tok<true, 4>; break;
    }
  }
  SST_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<grid, kV2Threads, smem, st>>>(t, out);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

// sst_upscale_blend writing raw-rgb24 bytes: K5's float32 result quantised
// as write_raw_video does (video.py:139-143), fused into the store -- the
// reference CLI's decode output (cli.py:181) without a float32 frame pass.
extern "C" int sst_upscale_blend_u8(const float* img, int G, int h, int w, int s, int H, int W,
                                    const SstPrevDesc* prev, int blend_n, uint8_t* out, void* stream) {
  if (G < 0 || h <= 0 || w <= 0 || H <= 0 || W <= 0) return SST_ERR_ARG;
  if (s != 2 && s != 3) return SST_ERR_ARG;
  if (H > h * s || W > w * s) return SST_ERR_ARG;
  if (blend_n < 1 || blend_n > 8) return SST_ERR_ARG;
  if (prev && blend_n > 4) return SST_ERR_UNSUPPORTED;
  if (G == 0) return SST_OK;
  if (!img || !out) return SST_ERR_ARG;
  if (G > 65535) return SST_ERR_ARG;
  UpArgs a{};
  a.img = img; a.G = G; a.h = h; a.w = w; a.s = s; a.H = H; a.W = W;
  a.prev = prev; a.n = blend_n; a.out8 = out;
  for (int i = 1; i <= 4; ++i) {
    a.alpha[i - 1] = (double)(blend_n - i) / (double)blend_n;
    a.beta[i - 1] = 1.0 - a.alpha[i - 1];
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // v2 (TMA windows, two samples per thread -> one 16-bit store per frame
  // row) when the working images admit a tensor map and rows are 2-byte
  // aligned; the one-sample-per-thread kernel otherwise
  CUtensorMap imap;
  memset(&imap, 0, sizeof(imap));
  const char* var = getenv("SST_K5_VARIANT");
  const bool four = (W * 3) % 4 == 0 && (reinterpret_cast<uintptr_t>(out) & 3u) == 0 && var &&
                    !strcmp(var, "u8f4");
  const bool v2 = var && !strcmp(var, "v2");
  // rows per CTA of the float32 kernel (SST_K5U8_BAND=16 / 32, A/B)
  const char* eb = getenv("SST_K5U8_BAND");
  const int ebv = eb ? atoi(eb) : kK5u8Band;
  const int band = (four || v2) ? 16 : (ebv == 16 || ebv == 48 ? ebv : 32);
  if (!(var && !strcmp(var, "v1")) && (W * 3) % 2 == 0 && (reinterpret_cast<uintptr_t>(out) & 1u) == 0 &&
      make_tmap_f32_3d(&imap, img, (uint64_t)w * 3, (uint64_t)h, (uint64_t)G * 2, kWF9,
                       band == 48 ? UpTmaSmem<48>::kWR : band == 32 ? UpTmaSmem<32>::kWR : UpTmaSmem<16>::kWR))
  {
    // two samples per thread (16-bit stores).  A/B: SST_K5_VARIANT=v2, the
    // exact float64 kernel (0.80 / 0.91 ms per 32 x 1080p GoPs, s=3 / 2);
    // u8f4, four samples per thread with 32-bit stores (needs rows 4-byte
    // aligned): 157 registers, 0.82 / 0.90 ms against 0.72 / 0.77 ms
    if (v2) return launch_k5_v2<16, uint8_t>(imap, a, prev, blend_n, st);
    if (four) return launch_k5_u8f<16, 4>(imap, a, prev, blend_n, st);
    if (band == 48) return launch_k5_u8f<48, 2>(imap, a, prev, blend_n, st);
    return band == 32 ? launch_k5_u8f<32, 2>(imap, a, prev, blend_n, st)
                      : launch_k5_u8f<16, 2>(imap, a, prev, blend_n, st);
  }
  dim3 grid(ceil_div(W * 3, kUpThreads), ceil_div(H, kUpRows), G);
  if (grid.y > 65535) return SST_ERR_ARG;
  k_upscale_blend<uint8_t><<<grid, kUpThreads, 0, st>>>(a);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_upscale_blend9(const float* img, int G, int h, int w, int s, int H, int W,
                                  const SstPrevDesc* prev, int blend_n, float* out, void* stream) {
  if (G < 0 || h <= 0 || w <= 0 || H <= 0 || W <= 0) return SST_ERR_ARG;
  if (s != 2 && s != 3) return SST_ERR_ARG;
  if (H > h * s || W > w * s) return SST_ERR_ARG;
  if (blend_n < 1 || blend_n > 8) return SST_ERR_ARG;
  if (prev && blend_n > 4) return SST_ERR_UNSUPPORTED;
  if (G == 0) return SST_OK;
  if (!img || !out || G > 65535) return SST_ERR_ARG;
  UpArgs a{};
  a.img = img; a.G = G; a.h = h; a.w = w; a.s = s; a.H = H; a.W = W;
  a.prev = prev; a.n = blend_n; a.out = out;
  for (int i = 1; i <= 4; ++i) {
    a.alpha[i - 1] = (double)(blend_n - i) / (double)blend_n;
    a.beta[i - 1] = 1.0 - a.alpha[i - 1];
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // Window loads: TMA boxes for the current GoP when its frames admit a
  // tensor map (16-byte aligned base and rows), else cp.async.  A/B switch:
  // SST_K5_9=sync | async | tma.  Measured (scripts/k5_9_micro.py, 32 x 1080p
  // GoPs, s=3, without / with blend n=2): register-staged loads 1.89 / 2.59 ms,
  // cp.async 1.49 / 2.12 ms.  Earlier layouts, since removed: one frame per
  // pass with TMA-store tiles 2.37 / 2.88 ms, column-private threads 3.0 / 4.1,
  // 32-row bands 2.24 / 3.28 (cp.async) and 3.5 / 4.8 (register-staged).
  // Window element type: float (default: 16-row bands, three CTAs per SM,
  // ~2 float32 <-> float64 conversions per output sample on the XU pipe) or
  // double (SST_K5_9W=f64: each source sample widened once, 12-row bands, two
  // CTAs per SM).  Measured (scripts/k5_9_micro.py, 32 x 1080p GoPs, s=3,
  // without / with blend): float 1.345 / 1.609 ms, double 1.959 / 2.331 ms --
  // the halved occupancy and the widening pass cost more than the XU work
  // they remove, so float stays the default.
  const char* ww = getenv("SST_K5_9W");
  const bool f32w = !(ww && !strcmp(ww, "f64"));
  constexpr int kB64 = 12, kB32 = 16;
  CUtensorMap imap;
  memset(&imap, 0, sizeof(imap));
  const bool tma_in = make_tmap_f32_3d(&imap, img, (uint64_t)w * 3, (uint64_t)h,
                                       (uint64_t)G * kGop, kWF9,
                                       f32w ? Up9fGeom<kB32>::kWR : Up9fGeom<kB64>::kWR);
  int load = tma_in ? 2 : 1;
  if (const char* v9 = getenv("SST_K5_9")) {
    if (!strcmp(v9, "sync")) load = 0;
    else if (!strcmp(v9, "async")) load = 1;
  }
  if (f32w) {
    if (load == 2) return launch_k5_9f<kB32, 2, float>(imap, a, prev, blend_n, st);
    if (load == 1) return launch_k5_9f<kB32, 1, float>(imap, a, prev, blend_n, st);
    return launch_k5_9f<kB32, 0, float>(imap, a, prev, blend_n, st);
  }
  if (load == 2) return launch_k5_9f<kB64, 2, double>(imap, a, prev, blend_n, st);
  if (load == 1) return launch_k5_9f<kB64, 1, double>(imap, a, prev, blend_n, st);
  return launch_k5_9f<kB64, 0, double>(imap, a, prev, blend_n, st);
}

extern "C" int sst_upscale(const float* img, int64_t n, int h, int w, int s, int crop_h, int crop_w,
                           float* out, void* stream) {
  if (n < 0 || h <= 0 || w <= 0 || crop_h <= 0 || crop_w <= 0) return SST_ERR_ARG;
  if (s != 2 && s != 3) return SST_ERR_ARG;
  if (crop_h > h * s || crop_w > w * s) return SST_ERR_ARG;
  if (n == 0) return SST_OK;
  if (!img || !out) return SST_ERR_ARG;
  int64_t total = n * crop_h * crop_w * 3;
  k_upscale<float, float, true><<<(unsigned)ceil_div64(total, 256), 256, 0,
                                  static_cast<cudaStream_t>(stream)>>>(img, n, h, w, s, crop_h,
                                                                       crop_w, out);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_bilinear_f64(const double* img, int64_t n, int h, int w, int s, double* out,
                                void* stream) {
  if (n < 0 || h <= 0 || w <= 0 || s <= 0) return SST_ERR_ARG;
  if (n == 0) return SST_OK;
  if (!img || !out) return SST_ERR_ARG;
  int64_t total = n * (int64_t)h * s * w * s * 3;
  k_upscale<double, double, false><<<(unsigned)ceil_div64(total, 256), 256, 0,
                                     static_cast<cudaStream_t>(stream)>>>(img, n, h, w, s, h * s,
                                                                          w * s, out);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_clip_cast(const double* x, int64_t count, float* out, void* stream) {
  if (count < 0) return SST_ERR_ARG;
  if (count == 0) return SST_OK;
  if (!x || !out) return SST_ERR_ARG;
  k_clip_cast<<<(unsigned)ceil_div64(count, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      x, count, out);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_blend(const float* prev, const float* curr, int G, int H, int W, int n, float* out,
                         void* stream) {
  if (G < 0 || H <= 0 || W <= 0) return SST_ERR_ARG;
  if (n < 1 || n > kGop) return SST_ERR_ARG;
  if (G == 0) return SST_OK;
  if (!prev || !curr || !out) return SST_ERR_ARG;
  int64_t fe = (int64_t)H * W * 3;
  k_blend<<<(unsigned)ceil_div64(G * fe, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      prev, curr, G, fe, n, out);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

// K5-9 over uint8 working frames q (sample value float(q / 255)): the int8
// learned tokenizer's decoder emits q directly (no float32 frames in HBM).
extern "C" int sst_upscale_blend9_u8(const uint8_t* img, int G, int h, int w, int s, int H, int W,
                                     const SstPrevDesc* prev, int blend_n, float* out,
                                     void* stream) {
  if (G < 0 || h <= 0 || w <= 0 || H <= 0 || W <= 0) return SST_ERR_ARG;
  if (s != 2 && s != 3) return SST_ERR_ARG;
  if (H > h * s || W > w * s) return SST_ERR_ARG;
  if (blend_n < 1 || blend_n > 8) return SST_ERR_ARG;
  if (prev && blend_n > 4) return SST_ERR_UNSUPPORTED;
  if (G == 0) return SST_OK;
  if (!img || !out || G > 65535) return SST_ERR_ARG;
  UpArgs a{};
  a.img = reinterpret_cast<const float*>(img); a.G = G; a.h = h; a.w = w; a.s = s; a.H = H; a.W = W;
  a.prev = prev; a.n = blend_n; a.out = out;
  for (int i = 1; i <= 4; ++i) {
    a.alpha[i - 1] = (double)(blend_n - i) / (double)blend_n;
    a.beta[i - 1] = 1.0 - a.alpha[i - 1];
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUtensorMap imap;
  memset(&imap, 0, sizeof(imap));
  // Output rows per CTA (SST_K59_U8_BAND=16|24|32|48|64 for A/B): byte
  // windows are small enough for 64-row bands, which amortise the per-CTA
  // setup (axis taps, window loads, LUT) over 4x the rows of the float
  // kernel's 16.  Measured (scripts/k5_9u8_micro.py, 32 x 1080p GoPs, s=3,
  // without / with blend n=2): 16 rows 1.500 / 1.696 ms, 32 rows 1.275 /
  // 1.490, 48 rows 1.240 / 1.452, 64 rows 1.257 / 1.416 (s=2: 1.903 / 2.091
  // -> 1.545 / 1.812).  With the 16-copy table (32 KB more per CTA) 48 rows
  // keep 3 CTAs per SM: s=3 1.216 / 1.361, s=2 1.325 / 1.637 ms.
  const char* bs = getenv("SST_K59_U8_BAND");
  const int band = bs ? atoi(bs) : (kLutC > 1 ? 48 : 64);
  auto go = [&](auto tag) -> int {
    constexpr int B = decltype(tag)::value;
    const bool t = make_tmap_u8_3d(&imap, img, (uint64_t)w * 3, (uint64_t)h, (uint64_t)G * kGop,
                                   kWF9u8, Up9fGeom<B, uint8_t>::kWR);
    // frames per pass when blending (the row-tap control repeats per pass,
    // registers hold 2 x frames float64 taps): measured with blend n=2, 48-row
    // bands (scripts/k5_9u8_micro.py, two runs) -- s=3: 5 + 4 1.320 ms, one
    // 9-frame pass 1.302, 3 + 6 1.311 (stable); s=2: 1.58-1.79 ms for every
    // split (run-to-run noise larger than the differences).  Default: one
    // pass at s=3, 5 + 4 at s=2; SST_K59_SPLIT=3|5|9 (A/B)
    const char* sp = getenv("SST_K59_SPLIT");
    const int split = sp ? atoi(sp) : (s == 3 ? 9 : 5);
    if (split == 9)
      return t ? launch_k5_9f<B, 2, uint8_t, 9>(imap, a, prev, blend_n, st)
               : launch_k5_9f<B, 0, uint8_t, 9>(imap, a, prev, blend_n, st);
    if (split == 3)
      return t ? launch_k5_9f<B, 2, uint8_t, 3>(imap, a, prev, blend_n, st)
               : launch_k5_9f<B, 0, uint8_t, 3>(imap, a, prev, blend_n, st);
    return t ? launch_k5_9f<B, 2, uint8_t>(imap, a, prev, blend_n, st)
             : launch_k5_9f<B, 0, uint8_t>(imap, a, prev, blend_n, st);
  };
  if (band == 24) return go(std::integral_constant<int, 24>{});
  if (band == 32) return go(std::integral_constant<int, 32>{});
  if (band == 40) return go(std::integral_constant<int, 40>{});
  if (band == 48) return go(std::integral_constant<int, 48>{});
  if (band == 64) return go(std::integral_constant<int, 64>{});
  const bool tma_in = make_tmap_u8_3d(&imap, img, (uint64_t)w * 3, (uint64_t)h, (uint64_t)G * kGop,
                                      kWF9u8, Up9fGeom<16, uint8_t>::kWR);
  if (tma_in) return launch_k5_9f<16, 2, uint8_t>(imap, a, prev, blend_n, st);
  return launch_k5_9f<16, 0, uint8_t>(imap, a, prev, blend_n, st);
}
