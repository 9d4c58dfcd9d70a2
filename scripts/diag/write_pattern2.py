"""Write-only DRAM rate of candidate K5 output orders (no compute): G GoPs x 9
frames of 1080p float32.  Variants: the K5 v2 band pattern (128 threads x
float2, 16-row bands, the 9 frames interleaved per row) at several band
heights, frame-outer order inside a band, float4 stores, and a contiguous
fill_ for reference.  Used to pick K5's store order."""
import torch
from torch.utils.cpp_extension import load_inline

src = r"""
#include <torch/extension.h>
// FO: frame-outer (all rows of frame f, then f+1) instead of row-outer
template <int VEC, int BAND, bool FO, int NT>
__global__ void __launch_bounds__(NT) k_bands(float* out, int H, int W3, int G) {
  const int q = (blockIdx.x * NT + threadIdx.x) * VEC;
  const int y0 = blockIdx.y * BAND, g = blockIdx.z;
  if (q >= W3) return;
  const long fs = (long)H * W3;
  float* base = out + (long)g * 9 * fs + (long)y0 * W3 + q;
  const int rows = min(BAND, H - y0);
  if (FO) {
    for (int f = 0; f < 9; ++f)
      for (int r = 0; r < rows; ++r) {
        float* o = base + f * fs + (long)r * W3;
        if (VEC == 2) __stcs(reinterpret_cast<float2*>(o), make_float2(0.5f, 0.5f));
        else __stcs(reinterpret_cast<float4*>(o), make_float4(0.5f, 0.5f, 0.5f, 0.5f));
      }
  } else {
    for (int r = 0; r < rows; ++r)
      for (int f = 0; f < 9; ++f) {
        float* o = base + f * fs + (long)r * W3;
        if (VEC == 2) __stcs(reinterpret_cast<float2*>(o), make_float2(0.5f, 0.5f));
        else __stcs(reinterpret_cast<float4*>(o), make_float4(0.5f, 0.5f, 0.5f, 0.5f));
      }
  }
}
// plain (non-streaming) stores
template <int BAND>
__global__ void __launch_bounds__(128) k_bands_wb(float* out, int H, int W3, int G) {
  const int q = (blockIdx.x * 128 + threadIdx.x) * 2;
  const int y0 = blockIdx.y * BAND, g = blockIdx.z;
  if (q >= W3) return;
  const long fs = (long)H * W3;
  float* base = out + (long)g * 9 * fs + (long)y0 * W3 + q;
  const int rows = min(BAND, H - y0);
  for (int r = 0; r < rows; ++r)
    for (int f = 0; f < 9; ++f)
      *reinterpret_cast<float2*>(base + f * fs + (long)r * W3) = make_float2(0.5f, 0.5f);
}
// K5's shape without its arithmetic: each CTA first stages its source
// windows (3 x 10 rows x 144 floats of a [G][2][540][960][3] image) in smem,
// then writes the band; kPF: the windows of the NEXT band are prefetched
// (persistent CTAs, double-buffered) so no CTA waits on a load
template <bool kPF>
__global__ void __launch_bounds__(128) k_load_store(float* out, const float* img, int H, int W3, int G,
                                                    int nitems) {
  __shared__ float win[2][3][10 * 144];
  const int ntx = (W3 / 2 + 127) / 128, nty = (H + 15) / 16;
  const long fs = (long)H * W3;
  const int h = 540, w3 = 2880;
  auto load = [&](int it, int b) {
    const int tx = it % ntx, ty = (it / ntx) % nty, g = it / (ntx * nty);
    const float* src = img + (long)g * 2 * h * w3 + (long)(ty * 8) * w3 + tx * 128;
    for (int i = threadIdx.x; i < 3 * 10 * 144; i += 128) {
      const int k = i / 1440, rr = (i % 1440) / 144, c = i % 144;
      const int row = min(ty * 8 + rr, h - 1);
      win[b][k][rr * 144 + c] = src[(long)(k == 2 ? 1 : k) * h * w3 + (long)(row - ty * 8) * w3 + min(c, w3 - 1 - tx * 128)];
    }
  };
  if (!kPF) {
    const int it = blockIdx.x;
    load(it, 0);
    __syncthreads();
    const int tx = it % ntx, ty = (it / ntx) % nty, g = it / (ntx * nty);
    const int q = (tx * 128 + threadIdx.x) * 2;
    if (q >= W3) return;
    float* base = out + (long)g * 9 * fs + (long)(ty * 16) * W3 + q;
    const int rows = min(16, H - ty * 16);
    for (int r = 0; r < rows; ++r) {
      const float v = win[0][0][(r / 2) * 144 + (threadIdx.x & 127)] + win[0][1][(r / 2) * 144 + 1] + win[0][2][5];
      for (int f = 0; f < 9; ++f)
        __stcs(reinterpret_cast<float2*>(base + f * fs + (long)r * W3), make_float2(v, v));
    }
    return;
  }
  int b = 0;
  int it = blockIdx.x;
  if (it < nitems) load(it, 0);
  for (; it < nitems; it += gridDim.x, b ^= 1) {
    __syncthreads();
    if (it + (int)gridDim.x < nitems) load(it + gridDim.x, b ^ 1);
    const int tx = it % ntx, ty = (it / ntx) % nty, g = it / (ntx * nty);
    const int q = (tx * 128 + threadIdx.x) * 2;
    if (q < W3) {
      float* base = out + (long)g * 9 * fs + (long)(ty * 16) * W3 + q;
      const int rows = min(16, H - ty * 16);
      for (int r = 0; r < rows; ++r) {
        const float v = win[b][0][(r / 2) * 144 + (threadIdx.x & 127)] + win[b][1][(r / 2) * 144 + 1] + win[b][2][5];
        for (int f = 0; f < 9; ++f)
          __stcs(reinterpret_cast<float2*>(base + f * fs + (long)r * W3), make_float2(v, v));
      }
    }
  }
}
void ldst(torch::Tensor out, torch::Tensor img, int64_t H, int64_t W3, int64_t G, int64_t pf, int64_t ctas) {
  const int n = (int)(((W3 / 2 + 127) / 128) * ((H + 15) / 16) * G);
  if (pf) k_load_store<true><<<(int)ctas, 128>>>(out.data_ptr<float>(), img.data_ptr<float>(), H, W3, G, n);
  else k_load_store<false><<<n, 128>>>(out.data_ptr<float>(), img.data_ptr<float>(), H, W3, G, n);
}
// frame-major: blockIdx.z = g * 9 + f, each CTA one frame's band
template <int BAND>
__global__ void __launch_bounds__(128) k_frame_major(float* out, int H, int W3) {
  const int q = (blockIdx.x * 128 + threadIdx.x) * 2;
  const int y0 = blockIdx.y * BAND;
  if (q >= W3) return;
  float* base = out + (long)blockIdx.z * H * W3 + (long)y0 * W3 + q;
  const int rows = min(BAND, H - y0);
  for (int r = 0; r < rows; ++r)
    __stcs(reinterpret_cast<float2*>(base + (long)r * W3), make_float2(0.5f, 0.5f));
}
// k frames per CTA: blockIdx.z = g * ceil(9/k) + j covers frames j*k .. j*k+k-1
template <int K>
__global__ void __launch_bounds__(128) k_frame_group(float* out, int H, int W3) {
  constexpr int NJ = (9 + K - 1) / K;
  const int q = (blockIdx.x * 128 + threadIdx.x) * 2;
  const int y0 = blockIdx.y * 16;
  if (q >= W3) return;
  const int g = blockIdx.z / NJ, j = blockIdx.z % NJ;
  const long fs = (long)H * W3;
  float* base = out + ((long)g * 9 + j * K) * fs + (long)y0 * W3 + q;
  const int rows = min(16, H - y0);
  const int nf = min(K, 9 - j * K);
  for (int r = 0; r < rows; ++r)
    for (int f = 0; f < nf; ++f)
      __stcs(reinterpret_cast<float2*>(base + f * fs + (long)r * W3), make_float2(0.5f, 0.5f));
}
// the band pattern preceded, in every CTA, by a coalesced float4 read of
// `rd` bytes at offset (CTA index * rd) modulo the source size (`wrap`):
// K5's DRAM read/write mix without its arithmetic
__global__ void __launch_bounds__(128) k_read_then_bands(float* out, const float4* src, long wrap4, int rd4,
                                                         int H, int W3) {
  __shared__ float4 buf[1536];
  const long cta = ((long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  const long off = (cta * rd4) % wrap4;
  for (int i = threadIdx.x; i < rd4; i += 128) buf[i] = src[off + i];
  __syncthreads();
  const int q = (blockIdx.x * 128 + threadIdx.x) * 2;
  const int y0 = blockIdx.y * 16, g = blockIdx.z;
  if (q >= W3) return;
  const long fs = (long)H * W3;
  float* base = out + (long)g * 9 * fs + (long)y0 * W3 + q;
  const int rows = min(16, H - y0);
  const float v = buf[threadIdx.x].x;
  for (int r = 0; r < rows; ++r)
    for (int f = 0; f < 9; ++f)
      __stcs(reinterpret_cast<float2*>(base + f * fs + (long)r * W3), make_float2(v, v));
}
// ... with the reads batched: every PF-th CTA bulk-prefetches into L2 the
// reads of the PF CTAs starting LA CTAs ahead (cp.async.bulk.prefetch.L2),
// so DRAM sees a few large read bursts instead of a read per CTA
__global__ void __launch_bounds__(128) k_read_then_bands_pf(float* out, const float4* src, long wrap4, int rd4,
                                                            int H, int W3, int pf, int la) {
  __shared__ float4 buf[1536];
  const long cta = ((long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  if (threadIdx.x == 0 && cta % pf == 0) {
    const long first = cta + la;
    for (long c = first; c < first + pf; c += 16) {
      const long o = (c * rd4) % wrap4;
      const long n = min((long)16 * rd4, wrap4 - o) * 16;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + o), "r"((unsigned)n) : "memory");
    }
  }
  const long off = (cta * rd4) % wrap4;
  for (int i = threadIdx.x; i < rd4; i += 128) buf[i] = src[off + i];
  __syncthreads();
  const int q = (blockIdx.x * 128 + threadIdx.x) * 2;
  const int y0 = blockIdx.y * 16, g = blockIdx.z;
  if (q >= W3) return;
  const long fs = (long)H * W3;
  float* base = out + (long)g * 9 * fs + (long)y0 * W3 + q;
  const int rows = min(16, H - y0);
  const float v = buf[threadIdx.x].x;
  for (int r = 0; r < rows; ++r)
    for (int f = 0; f < 9; ++f)
      __stcs(reinterpret_cast<float2*>(base + f * fs + (long)r * W3), make_float2(v, v));
}
void rdbpf(torch::Tensor out, torch::Tensor src, int64_t H, int64_t W3, int64_t G, int64_t rd_bytes,
           int64_t wrap_bytes, int64_t pf, int64_t la) {
  dim3 grid((W3 / 2 + 127) / 128, (H + 15) / 16, G);
  k_read_then_bands_pf<<<grid, 128>>>(out.data_ptr<float>(), reinterpret_cast<const float4*>(src.data_ptr<float>()),
                                      wrap_bytes / 16, (int)(rd_bytes / 16), H, W3, (int)pf, (int)la);
}
void rdb(torch::Tensor out, torch::Tensor src, int64_t H, int64_t W3, int64_t G, int64_t rd_bytes, int64_t wrap_bytes) {
  dim3 grid((W3 / 2 + 127) / 128, (H + 15) / 16, G);
  k_read_then_bands<<<grid, 128>>>(out.data_ptr<float>(), reinterpret_cast<const float4*>(src.data_ptr<float>()),
                                   wrap_bytes / 16, (int)(rd_bytes / 16), H, W3);
}
void fgrp(torch::Tensor out, int64_t H, int64_t W3, int64_t G, int64_t k) {
  dim3 grid((W3 / 2 + 127) / 128, (H + 15) / 16, 1);
  if (k == 2) { grid.z = G * 5; k_frame_group<2><<<grid, 128>>>(out.data_ptr<float>(), H, W3); }
  if (k == 3) { grid.z = G * 3; k_frame_group<3><<<grid, 128>>>(out.data_ptr<float>(), H, W3); }
  if (k == 5) { grid.z = G * 2; k_frame_group<5><<<grid, 128>>>(out.data_ptr<float>(), H, W3); }
}
void fmaj(torch::Tensor out, int64_t H, int64_t W3, int64_t G, int64_t band) {
  if (band == 16) {
    dim3 grid((W3 / 2 + 127) / 128, (H + 15) / 16, G * 9);
    k_frame_major<16><<<grid, 128>>>(out.data_ptr<float>(), H, W3);
  } else if (band == 32) {
    dim3 grid((W3 / 2 + 127) / 128, (H + 31) / 32, G * 9);
    k_frame_major<32><<<grid, 128>>>(out.data_ptr<float>(), H, W3);
  } else {
    dim3 grid((W3 / 2 + 127) / 128, (H + 63) / 64, G * 9);
    k_frame_major<64><<<grid, 128>>>(out.data_ptr<float>(), H, W3);
  }
}
template <int VEC, int BAND, bool FO, int NT>
void go(torch::Tensor out, int H, int W3, int G) {
  dim3 grid((W3 / VEC + NT - 1) / NT, (H + BAND - 1) / BAND, G);
  k_bands<VEC, BAND, FO, NT><<<grid, NT>>>(out.data_ptr<float>(), H, W3, G);
}
void bands(torch::Tensor out, int64_t H, int64_t W3, int64_t G, int64_t v) {
  switch (v) {
    case 0: go<2, 16, false, 128>(out, H, W3, G); break;   // K5 v2 pattern
    case 1: go<2, 8, false, 128>(out, H, W3, G); break;
    case 2: go<2, 32, false, 128>(out, H, W3, G); break;
    case 3: go<2, 64, false, 128>(out, H, W3, G); break;
    case 4: go<2, 16, true, 128>(out, H, W3, G); break;
    case 5: go<4, 16, false, 128>(out, H, W3, G); break;
    case 6: go<2, 16, false, 256>(out, H, W3, G); break;
    case 7: go<2, 16, false, 64>(out, H, W3, G); break;
    case 8: go<4, 32, false, 64>(out, H, W3, G); break;
    case 9: { dim3 grid((W3 / 2 + 127) / 128, (H + 15) / 16, G);
              k_bands_wb<16><<<grid, 128>>>(out.data_ptr<float>(), H, W3, G); break; }
  }
}
"""
m = load_inline("wpat2", cpp_sources="void bands(torch::Tensor out, int64_t H, int64_t W3, int64_t G, int64_t v);"
                "void ldst(torch::Tensor out, torch::Tensor img, int64_t H, int64_t W3, int64_t G, int64_t pf, int64_t ctas);"
                "void fmaj(torch::Tensor out, int64_t H, int64_t W3, int64_t G, int64_t band);"
                "void fgrp(torch::Tensor out, int64_t H, int64_t W3, int64_t G, int64_t k);"
                "void rdb(torch::Tensor out, torch::Tensor src, int64_t H, int64_t W3, int64_t G, int64_t rd_bytes, int64_t wrap_bytes);"
                "void rdbpf(torch::Tensor out, torch::Tensor src, int64_t H, int64_t W3, int64_t G, int64_t rd_bytes, int64_t wrap_bytes, int64_t pf, int64_t la);",
                cuda_sources=src, functions=["bands", "ldst", "fmaj", "fgrp", "rdb", "rdbpf"],
                extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"])
G, H, W = 32, 1080, 1920
out = torch.empty((G, 9, H, W, 3), device="cuda")
img = torch.rand((G, 2, 540, 960, 3), device="cuda")
nbytes = out.numel() * 4
names = ["v2 pattern: float2 x 128 thr, band 16, row-outer", "band 8", "band 32", "band 64",
         "band 16 frame-outer", "float4 x 128 thr band 16", "float2 x 256 thr band 16",
         "float2 x 64 thr band 16", "float4 x 64 thr band 32", "band 16 write-back (st.global)"]


def t(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


src_big = torch.rand(64 << 20, device="cuda")      # 256 MB: reads come from DRAM
import sys
if "--reads" in sys.argv:
    for rep in range(2):
        ms = t(lambda: m.bands(out, H, W * 3, G, 0))
        print(f"{'band pattern, no reads':48s}: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s")
        for rd in (3584,):
            for wrap in (1 << 20, 256 << 20):
                ms = t(lambda: m.rdb(out, src_big, H, W * 3, G, rd, wrap))
                print(f"{'+ %d B read per CTA from %d MB' % (rd, wrap >> 20):48s}: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s")
            for pf in (64, 256, 1024):
                for la in (1024, 4096):
                    ms = t(lambda: m.rdbpf(out, src_big, H, W * 3, G, rd, 256 << 20, pf, la))
                    print(f"{'  L2 bulk prefetch: every %d CTAs, %d ahead' % (pf, la):48s}: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s")
    sys.exit(0)
for rep in range(2):
    for v, nm in enumerate(names):
        ms = t(lambda: m.bands(out, H, W * 3, G, v))
        print(f"{nm:48s}: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s")
    ms = t(lambda: out.fill_(0.5))
    print(f"{'contiguous fill_':48s}: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s")
    for band in (16, 32, 64):
        ms = t(lambda: m.fmaj(out, H, W * 3, G, band))
        print(f"{'frame-major CTAs, band %d' % band:48s}: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s")
    for k in (2, 3, 5):
        ms = t(lambda: m.fgrp(out, H, W * 3, G, k))
        print(f"{'%d frames per CTA, band 16' % k:48s}: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s")
    ms = t(lambda: m.ldst(out, img, H, W * 3, G, 0, 0))
    print(f"{'load windows, then store (one band per CTA)':48s}: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s")
    for k in (4, 6, 8, 12):
        ms = t(lambda: m.ldst(out, img, H, W * 3, G, 1, 148 * k))
        print(f"{'persistent, next window prefetched, %d/SM' % k:48s}: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s")
