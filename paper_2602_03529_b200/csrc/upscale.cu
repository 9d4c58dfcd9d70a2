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
#include "common.cuh"

namespace sst {

struct AxisTap {
  int lo, hi;
  double f, g;   // frac, 1 - frac
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

__device__ __forceinline__ float blend_px(float prev, float curr, double alpha) {
  double v = alpha * (double)prev + (1.0 - alpha) * (double)curr;   // codec.py:293
  return (float)clip01(v);
}

// ---- fused upscale + blend + 9-frame store ----
constexpr int kUpRows = 8;
constexpr int kUpCols = 64;
constexpr int kUpThreads = 256;

struct UpArgs {
  const float* img;            // [G][2][h][w][3]
  int G, h, w, s, H, W;
  const SstPrevDesc* prev;     // [G] or null
  int n;                       // blend width
  float* out;                  // [G][9][H][W][3]
};

__global__ void __launch_bounds__(kUpThreads) k_upscale_blend(UpArgs a) {
  __shared__ AxisTap ty_c[kUpRows], tx_c[kUpCols];
  __shared__ AxisTap ty_p[kUpRows], tx_p[kUpCols];
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * kUpCols;
  const int y0 = blockIdx.y * kUpRows;
  const int g = blockIdx.z;
  SstPrevDesc pd;
  pd.p_img = nullptr;
  if (a.prev) pd = a.prev[g];
  const bool has_prev = pd.p_img != nullptr;
  if (tid < kUpRows) ty_c[tid] = axis_tap(y0 + tid, a.h, a.s);
  else if (tid < kUpRows + kUpCols) tx_c[tid - kUpRows] = axis_tap(x0 + tid - kUpRows, a.w, a.s);
  else if (has_prev && tid < 2 * kUpRows + kUpCols) ty_p[tid - kUpRows - kUpCols] =
      axis_tap(y0 + tid - kUpRows - kUpCols, pd.h, pd.s);
  else if (has_prev && tid >= 128 && tid < 128 + kUpCols)
    tx_p[tid - 128] = axis_tap(x0 + tid - 128, pd.w, pd.s);
  __syncthreads();

  const float* iimg = a.img + (int64_t)g * 2 * a.h * a.w * 3;
  const float* pimg = iimg + (int64_t)a.h * a.w * 3;
  const int64_t fstride = (int64_t)a.H * a.W * 3;
  float* og = a.out + (int64_t)g * kGop * fstride;
  const int rows = min(kUpRows, a.H - y0);
  const int cols = min(kUpCols, a.W - x0);
  for (int e = tid; e < kUpRows * kUpCols * 3; e += kUpThreads) {
    const int r = e / (kUpCols * 3);
    const int q = e % (kUpCols * 3);
    const int px = q / 3, ch = q % 3;
    if (r >= rows || px >= cols) continue;
    const float ui = (float)clip01(bilerp(iimg, a.w, ty_c[r], tx_c[px], ch));
    const float up = (float)clip01(bilerp(pimg, a.w, ty_c[r], tx_c[px], ch));
    float* o = og + ((int64_t)(y0 + r) * a.W + x0) * 3 + q;
    if (has_prev) {
      const float uq = (float)clip01(bilerp(pd.p_img, pd.w, ty_p[r], tx_p[px], ch));
      // frame f < n: i = f + 1, alpha = (n - i) / n, prev frame 9 - n + f (= uq)
      __stcs(o, blend_px(uq, ui, (double)(a.n - 1) / (double)a.n));
      for (int f = 1; f < kGop; ++f)
        __stcs(o + f * fstride, f < a.n ? blend_px(uq, up, (double)(a.n - 1 - f) / (double)a.n) : up);
    } else {
      __stcs(o, ui);
#pragma unroll
      for (int f = 1; f < kGop; ++f) __stcs(o + f * fstride, up);
    }
  }
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

constexpr int kMseThreads = 512;

__global__ void __launch_bounds__(kMseThreads)
    k_mse(const float* __restrict__ a, const float* __restrict__ b, int64_t elems, double* out) {
  __shared__ double part[kMseThreads / 32];
  const float* pa = a + (int64_t)blockIdx.x * elems;
  const float* pb = b + (int64_t)blockIdx.x * elems;
  double acc = 0.0;
  for (int64_t e = threadIdx.x; e < elems; e += kMseThreads) {
    double d = (double)pa[e] - (double)pb[e];
    acc = acc + d * d;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < kMseThreads / 32; ++i) s += part[i];
    out[blockIdx.x] = s / (double)elems;
  }
}

}  // namespace sst

using namespace sst;

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
  UpArgs a{img, G, h, w, s, H, W, prev, blend_n, out};
  dim3 grid(ceil_div(W, kUpCols), ceil_div(H, kUpRows), G);
  if (grid.y > 65535) return SST_ERR_ARG;
  k_upscale_blend<<<grid, kUpThreads, 0, static_cast<cudaStream_t>(stream)>>>(a);
  SST_LAUNCH_CHECK();
  return SST_OK;
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

extern "C" int sst_mse(const float* a, const float* b, int64_t n, int64_t elems, double* out,
                       void* stream) {
  if (n < 0 || elems <= 0) return SST_ERR_ARG;
  if (n == 0) return SST_OK;
  if (!a || !b || !out) return SST_ERR_ARG;
  k_mse<<<(unsigned)n, kMseThreads, 0, static_cast<cudaStream_t>(stream)>>>(a, b, elems, out);
  SST_LAUNCH_CHECK();
  return SST_OK;
}
