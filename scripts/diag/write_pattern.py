"""Write-only DRAM rate of K5's output pattern (no compute): G GoPs x 9 frames
of 1080p float32, each CTA a 16-row band x SEG contiguous bytes per row and
frame (the real K5 uses 1 KB segments), vs a plain contiguous fill."""
import torch
from torch.utils.cpp_extension import load_inline

src = r"""
#include <torch/extension.h>
template <int VEC>
__global__ void k_bands(float* out, int H, int W3, int G) {
  // blockIdx.x: column tile of 256*VEC floats, y: 16-row band, z: GoP
  const int q = (blockIdx.x * 256 + threadIdx.x) * VEC;
  const int y0 = blockIdx.y * 16, g = blockIdx.z;
  if (q >= W3) return;
  const long fs = (long)H * W3;
  for (int r = 0; r < 16 && y0 + r < H; ++r) {
    float* o = out + (long)g * 9 * fs + (long)(y0 + r) * W3 + q;
    for (int f = 0; f < 9; ++f) {
      if (VEC == 1) __stcs(o + f * fs, 0.5f);
      else if (VEC == 2) __stcs(reinterpret_cast<float2*>(o + f * fs), make_float2(0.5f, 0.5f));
      else __stcs(reinterpret_cast<float4*>(o + f * fs), make_float4(0.5f, 0.5f, 0.5f, 0.5f));
    }
  }
}
void bands(torch::Tensor out, int64_t H, int64_t W3, int64_t G, int64_t vec) {
  dim3 grid((W3 / vec + 255) / 256, (H + 15) / 16, G);
  if (vec == 1) k_bands<1><<<grid, 256>>>(out.data_ptr<float>(), H, W3, G);
  else if (vec == 2) k_bands<2><<<grid, 256>>>(out.data_ptr<float>(), H, W3, G);
  else k_bands<4><<<grid, 256>>>(out.data_ptr<float>(), H, W3, G);
}
"""
m = load_inline("wpat", cpp_sources="void bands(torch::Tensor out, int64_t H, int64_t W3, int64_t G, int64_t vec);",
                cuda_sources=src, functions=["bands"],
                extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"])
G, H, W = 32, 1080, 1920
out = torch.empty((G, 9, H, W, 3), device="cuda")
nbytes = out.numel() * 4


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


for vec in (1, 2, 4):
    ms = t(lambda: m.bands(out, H, W * 3, G, vec))
    print(f"bands, {256 * vec * 4} B segments: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s")
ms = t(lambda: out.fill_(0.5))
print(f"contiguous fill_: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s")
