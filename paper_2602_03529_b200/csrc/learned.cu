// Learned-tokenizer plug-in kernels: a causal
// spatio-temporal convolutional tokenizer with finite-scalar quantisation,
// plugged in at the reference's tokenizer hook (session.py:57-61).
//
//   k_lt_patchify  box downscale (bit-exact, codec.py:202-214) + edge pad to
//                  the 8x8 grid (codec.py:99-105) + 8x8(x8) patchify -> bf16
//   k_lt_conv      implicit-GEMM convolution on the 5th-gen tensor cores:
//                  one CTA computes a 128-token x BN-channel tile.  Warp 0
//                  (one lane) streams A (the im2col view of the activation,
//                  fetched per tap by 5-D TMA with zero-filled halo) and B
//                  (weights) into a 4-stage 128B-swizzled smem ring; warp 1
//                  (one lane) issues tcgen05.mma (M=128, N=BN, K=16) into a
//                  TMEM accumulator; then all four warps drain TMEM with
//                  tcgen05.ld and run the fused epilogue:
//                    STORE   +bias, SiLU, +residual -> bf16 -> TMA store
//                    FSQ     +bias, FSQ bound/round, codes f64 + indices
//                    PIXELS  +bias, clamp, depth-to-space f32 frame stores
//   k_lt_dec_in    mask-aware decoder input (snap to the FSQ grid, conceal
//                  masked P tokens with the co-located I token)
//
// The reference ships no learned model, so there is nothing to
// match bit-for-bit; oracle/learned_oracle.py restates the same network in
// torch fp32 with the same bf16 rounding points (parity unpinned).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstring>

#include "common.cuh"
#include "tc.cuh"

namespace sst {
namespace lt {

constexpr int BM = 128;            // tokens per tile (16 x 8 spatial box)
constexpr int BOX_X = 16, BOX_Y = 8;
constexpr int BK = 64;             // bf16 per 128-byte swizzled row
constexpr int A_BYTES = BM * BK * 2;
constexpr int FSQ_C = 12;          // 2 groups x levels (8,8,8,5,5,5)
constexpr int DEC_IN_C = 64;

__device__ __forceinline__ int fsq_levels(int i) { return (i % 6) < 3 ? 8 : 5; }
__device__ __forceinline__ int fsq_basis(int i) {
  // mixed radix inside one 6-dim group: 1, 8, 64, 512, 2560, 12800
  const int j = i % 6;
  return j == 0 ? 1 : j == 1 ? 8 : j == 2 ? 64 : j == 3 ? 512 : j == 4 ? 2560 : 12800;
}

struct ConvArgs {
  int Ht, Wt, tiles_x, tiles_y, t_lo, t_cnt;
  int n_taps, kb_per_tap, N, out_T;
  signed char taps[27][3];
  const float* bias;
  int act;
  const __nv_bfloat16* residual;
  __nv_bfloat16* out;          // STORE output of the halo / CTA-pair kernels (direct stores)
  double* codes;
  int32_t* idx;
  uint8_t* mask;
  float* frames;
  int h, w, frame_base;
};

__device__ __forceinline__ float silu(float x) { return __fdividef(x, 1.0f + __expf(-x)); }

// +bf16 residual for 32 channels at element offset off (STORE epilogues)
__device__ __forceinline__ void epi_add_residual(float (&v)[32], const ConvArgs& a, size_t off) {
  if (a.residual == nullptr) return;
  const uint4* rp = reinterpret_cast<const uint4*>(a.residual + off);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u = __ldg(rp + q);
    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 f = __bfloat1622float2(h2[e]);
      v[q * 8 + 2 * e] += f.x;
      v[q * 8 + 2 * e + 1] += f.y;
    }
  }
}

template <int BN, int NST>
struct TileCfg {
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  static constexpr int SMEM = NST * STAGE_BYTES + 1024 + 256;
};

// NST = smem pipeline stages: 4 for long K, 2 for the short-K (<= 512) 1x1
// layers so that 2-3 CTAs share an SM and one CTA's epilogue overlaps
// another's loads and MMAs.
template <int BN, int EPI, int NST>
__global__ void __launch_bounds__(128)
    k_lt_conv(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmC, const ConvArgs a) {
  constexpr int STAGES = NST;
  using Cfg = TileCfg<BN, NST>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * Cfg::B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* accum = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const int warp = threadIdx.x >> 5;
  int tile = blockIdx.x;
  const int tx = tile % a.tiles_x; tile /= a.tiles_x;
  const int ty = tile % a.tiles_y; tile /= a.tiles_y;
  const int t = a.t_lo + tile % a.t_cnt;
  const int g = tile / a.t_cnt;
  const int x0 = tx * BOX_X, y0 = ty * BOX_Y;
  const int n0 = blockIdx.y * BN;

  if (threadIdx.x == 0) {
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
    if (EPI == SST_LT_EPI_STORE) tc::prefetch_tmap(&tmC);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum, 1);
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  const int nkb = a.n_taps * a.kb_per_tap;
  if (threadIdx.x == 0) {
    // ---- TMA producer ----
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
      const int tap = kb / a.kb_per_tap, cb = kb - tap * a.kb_per_tap;
      mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
      tc::tma_load_5d(sA + s * A_BYTES, &tmA, cb * BK, x0 + a.taps[tap][2], y0 + a.taps[tap][1],
                      t + a.taps[tap][0], g, &full[s]);
      tc::tma_load_2d(sB + s * Cfg::B_BYTES, &tmB, kb * BK, n0, &full[s]);
    }
  } else if (threadIdx.x == 32) {
    // ---- MMA issuer ----
    constexpr uint32_t idesc = tc::idesc_bf16_f32(BM, BN);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      tc::fence_after_sync();
      const uint64_t ad = tc::smem_desc_sw128(smem_u32(sA + s * A_BYTES));
      const uint64_t bd = tc::smem_desc_sw128(smem_u32(sB + s * Cfg::B_BYTES));
#pragma unroll
      for (int k = 0; k < BK / 16; ++k)  // +32 B along K inside the swizzle atom
        tc::mma_bf16(tmem, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
      tc::mma_commit(&empty[s]);
    }
    tc::mma_commit(accum);
  }
  __syncwarp();
  mbar_wait(accum, 0);
  tc::fence_after_sync();

  // ---- epilogue: thread r owns accumulator row r (TMEM lane r) ----
  const int r = threadIdx.x;
  const int y = y0 + (r >> 4), x = x0 + (r & 15);
  const bool valid = y < a.Ht && x < a.Wt;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);

  if constexpr (EPI == SST_LT_EPI_STORE) {
    uint8_t* stage = sA;  // all loads consumed: reuse the A ring as the store tile
    const size_t tok = (((size_t)g * a.out_T + t) * a.Ht + y) * a.Wt + x;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      float v[32];
      tc::tmem_ld32(trow + c, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        v[i] += __ldg(a.bias + n0 + c + i);
        if (a.act) v[i] = silu(v[i]);
      }
      if (a.residual != nullptr && valid) {
        const uint4* rp = reinterpret_cast<const uint4*>(a.residual + tok * a.N + n0 + c);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u = __ldg(rp + q);
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float2 f = __bfloat1622float2(h2[e]);
            v[q * 8 + 2 * e] += f.x;
            v[q * 8 + 2 * e + 1] += f.y;
          }
        }
      }
      const int box = c >> 6, j0 = (c & 63) >> 3;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 u;
        __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) h2[e] = __floats2bfloat162_rn(v[q * 8 + 2 * e], v[q * 8 + 2 * e + 1]);
        const int j = j0 + q;
        *reinterpret_cast<uint4*>(stage + box * A_BYTES + r * 128 + ((j ^ (r & 7)) << 4)) = u;
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int b = 0; b < BN / 64; ++b) tc::tma_store_5d(&tmC, stage + b * A_BYTES, n0 + b * 64, x0, y0, t, g);
      tma_store_commit();
      tma_store_wait_all();
    }
  } else if constexpr (EPI == SST_LT_EPI_FSQ) {
    float v[16];
    tc::tmem_ld16(trow, v);
    if (valid) {
      const size_t tok = (((size_t)g * 2 + t) * a.Ht + y) * a.Wt + x;
      double codes[FSQ_C];
      int idx0 = 0, idx1 = 0;
#pragma unroll
      for (int i = 0; i < FSQ_C; ++i) {
        const int L = fsq_levels(i);
        // constants rounded once from float64, exactly as the oracle does
        const float half_l = (float)((double)(L - 1) * (1.0 - 1e-3) * 0.5);
        const float offset = (L % 2 == 0) ? 0.5f : 0.0f;
        const float shift = (float)atanh((double)offset / (double)half_l);
        const float z = v[i] + __ldg(a.bias + i);
        const float b = tanhf(z + shift) * half_l - offset;
        const int q = (int)rintf(b);
        const int hw = L / 2;
        codes[i] = (double)q / (double)hw;
        const int digit = (q + hw) * fsq_basis(i);
        if (i < 6) idx0 += digit; else idx1 += digit;
      }
      double2* cp = reinterpret_cast<double2*>(a.codes + tok * FSQ_C);
#pragma unroll
      for (int i = 0; i < FSQ_C / 2; ++i) cp[i] = make_double2(codes[2 * i], codes[2 * i + 1]);
      reinterpret_cast<int2*>(a.idx)[tok] = make_int2(idx0, idx1);
      a.mask[tok] = 1;
    }
  } else {  // SST_LT_EPI_PIXELS: 192 columns = one frame's 8x8x3 patch
    const int f = a.frame_base + blockIdx.y;
    const bool vec = (a.w & 3) == 0;
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
      float v[96];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        float u[32];
        tc::tmem_ld32(trow + half * 96 + q * 32, u);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[q * 32 + i] = u[i];
      }
      if (!valid) continue;
#pragma unroll
      for (int i = 0; i < 96; ++i)
        v[i] = fminf(fmaxf(v[i] + __ldg(a.bias + n0 + half * 96 + i), 0.0f), 1.0f);
#pragma unroll
      for (int pr = 0; pr < 4; ++pr) {
        const int Y = y * 8 + half * 4 + pr;
        if (Y >= a.h) continue;
        const int X0 = x * 8;
        float* dst = a.frames + ((((size_t)g * 9 + f) * a.h + Y) * a.w + X0) * 3;
        if (vec && X0 + 8 <= a.w) {
          float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
          for (int e = 0; e < 6; ++e)
            d4[e] = make_float4(v[pr * 24 + 4 * e], v[pr * 24 + 4 * e + 1], v[pr * 24 + 4 * e + 2],
                                v[pr * 24 + 4 * e + 3]);
        } else {
          const int npx = min(8, a.w - X0);
#pragma unroll
          for (int e = 0; e < 24; ++e)
            if (e / 3 < npx) dst[e] = v[pr * 24 + e];
        }
      }
    }
  }

  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, Cfg::TMEM_COLS);
}

// ---- causal (2,3,3) convolution with halo reuse ----------------------------
// A CTA computes 256 tokens (a 16 x 16 spatial tile of one latent frame) x 256
// output channels as two M=128 tcgen05 accumulators (TMEM columns 0..255 and
// 256..511).  For each (temporal tap, 64-channel block) ONE 5-D TMA box brings
// the tile's 18 x 18 halo (zero-filled outside the frame and
// before t=0) into shared memory; the nine spatial taps are then nine UMMA
// descriptors into that halo (start row (1+dy)*18 + (1+dx) [+ 8 for the right
// half], 8-row groups 18 rows apart), so A is fetched once per 9 taps instead
// of 9 times.  The 128-byte swizzle is a function of the absolute shared
// address for both TMA and UMMA, so descriptors may start on any 128-byte row
// (base offset 0) and the group stride need not be a multiple of 1024 B.  The weights stream through a 3-stage ring, each B stage feeding
// 2 x 4 MMAs.  L2->SM traffic per 256 tokens: 8 halos x 41 KB + the weights
// once (2.36 MB), vs 2 x 18 x 16 KB x 4 + 2 x 2.36 MB for the generic kernel.
namespace c233 {
constexpr int TILE = 16;                // 16 x 16 output tokens
constexpr int PITCH = 18;               // halo row pitch in tokens (dense: the swizzle is on absolute smem addresses)
constexpr int HROWS = 18;               // halo rows
constexpr int HALO_BYTES = PITCH * HROWS * 128;   // 41472
constexpr int BN = 256;
constexpr int B_BYTES = BN * 128;       // 32768
constexpr int HALO_STRIDE = (HALO_BYTES + 1023) / 1024 * 1024;  // slots stay 1024-B aligned
constexpr int HSLOTS = 2, BSTAGES = 4;
constexpr int SMEM = HSLOTS * HALO_STRIDE + BSTAGES * B_BYTES + 1024 + 256;
constexpr int THREADS = 256;
}  // namespace c233

__device__ __forceinline__ uint64_t halo_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((c233::PITCH * 128) >> 4) << 32;   // 8-row groups are PITCH rows apart
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__global__ void __launch_bounds__(c233::THREADS, 1)
    k_lt_conv233(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const ConvArgs a) {
  using namespace c233;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sH = smem;
  uint8_t* sB = smem + HSLOTS * HALO_STRIDE;
  uint64_t* hfull = reinterpret_cast<uint64_t*>(sB + BSTAGES * B_BYTES);
  uint64_t* hempty = hfull + HSLOTS;
  uint64_t* bfull = hempty + HSLOTS;
  uint64_t* bempty = bfull + BSTAGES;
  uint64_t* accum = bempty + BSTAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const int warp = threadIdx.x >> 5;
  int tile = blockIdx.x;
  const int tx = tile % a.tiles_x; tile /= a.tiles_x;
  const int ty = tile % a.tiles_y; tile /= a.tiles_y;
  const int t = a.t_lo + tile % a.t_cnt;
  const int g = tile / a.t_cnt;
  const int x0 = tx * TILE, y0 = ty * TILE;
  const int n0 = blockIdx.y * BN;

  if (threadIdx.x == 0) {
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
    for (int i = 0; i < HSLOTS; ++i) { mbar_init(&hfull[i], 1); mbar_init(&hempty[i], 1); }
    for (int i = 0; i < BSTAGES; ++i) { mbar_init(&bfull[i], 1); mbar_init(&bempty[i], 1); }
    mbar_init(accum, 1);
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  const int nh = 2 * a.kb_per_tap;   // (temporal tap, channel block) pairs
  const int C = a.kb_per_tap * BK;
  if (threadIdx.x == 0) {
    // ---- TMA producer: halos and weight k-blocks in consumption order ----
    int kb = 0;
    for (int hi = 0; hi < nh; ++hi) {
      const int kt = hi / a.kb_per_tap, cb = hi - kt * a.kb_per_tap;
      const int hs = hi % HSLOTS;
      if (hi >= HSLOTS) mbar_wait(&hempty[hs], ((hi / HSLOTS) - 1) & 1);
      mbar_expect_tx(&hfull[hs], HALO_BYTES);
      tc::tma_load_5d(sH + hs * HALO_STRIDE, &tmA, cb * BK, x0 - 1, y0 - 1, t + kt - 1, g, &hfull[hs]);
      for (int sp = 0; sp < 9; ++sp, ++kb) {
        const int bs = kb % BSTAGES;
        if (kb >= BSTAGES) mbar_wait(&bempty[bs], ((kb / BSTAGES) - 1) & 1);
        mbar_expect_tx(&bfull[bs], B_BYTES);
        const int tap = kt * 9 + sp;
        tc::tma_load_2d(sB + bs * B_BYTES, &tmB, tap * C + cb * BK, n0, &bfull[bs]);
      }
    }
  } else if (threadIdx.x == 32) {
    // ---- MMA issuer ----
    constexpr uint32_t idesc = tc::idesc_bf16_f32(128, BN);
    int kb = 0;
    for (int hi = 0; hi < nh; ++hi) {
      const int hs = hi % HSLOTS;
      mbar_wait(&hfull[hs], (hi / HSLOTS) & 1);
      const uint32_t hbase = smem_u32(sH + hs * HALO_STRIDE);
      for (int sp = 0; sp < 9; ++sp, ++kb) {
        const int bs = kb % BSTAGES;
        mbar_wait(&bfull[bs], (kb / BSTAGES) & 1);
        tc::fence_after_sync();
        const int dy = sp / 3, dx = sp % 3;   // halo offsets (1+dy', 1+dx')
        const uint64_t bd = tc::smem_desc_sw128(smem_u32(sB + bs * B_BYTES));
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const uint64_t ad = halo_desc(hbase + (uint32_t)((dy * PITCH + dx + 8 * half) * 128));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            tc::mma_bf16(tmem + half * BN, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
        }
        tc::mma_commit(&bempty[bs]);
      }
      tc::mma_commit(&hempty[hs]);
    }
    tc::mma_commit(accum);
  }
  __syncwarp();
  mbar_wait(accum, 0);
  tc::fence_after_sync();

  // ---- epilogue: 8 warps; warp w drains half (w >> 2), TMEM lanes 32*(w & 3) ----
  const int half = warp >> 2, q = warp & 3;
  const int m = q * 32 + (threadIdx.x & 31);        // accumulator row
  const int y = y0 + (m >> 3), x = x0 + half * 8 + (m & 7);
  const bool valid = y < a.Ht && x < a.Wt;
  const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + half * BN;
  const size_t tok = (((size_t)g * a.out_T + t) * a.Ht + y) * a.Wt + x;
  __nv_bfloat16* outp = a.out + tok * a.N + n0;
#pragma unroll 1
  for (int c = 0; c < BN; c += 32) {
    float v[32];
    tc::tmem_ld32(trow + c, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      v[i] += __ldg(a.bias + n0 + c + i);
      if (a.act) v[i] = silu(v[i]);
    }
    if (!valid) continue;
    if (a.residual != nullptr) {
      const uint4* rp = reinterpret_cast<const uint4*>(a.residual + tok * a.N + n0 + c);
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) {
        uint4 u = __ldg(rp + qq);
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 f = __bfloat1622float2(h2[e]);
          v[qq * 8 + 2 * e] += f.x;
          v[qq * 8 + 2 * e + 1] += f.y;
        }
      }
    }
    uint4* op = reinterpret_cast<uint4*>(outp + c);
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      uint4 u;
      __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) h2[e] = __floats2bfloat162_rn(v[qq * 8 + 2 * e], v[qq * 8 + 2 * e + 1]);
      op[qq] = u;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// ---- persistent, warp-specialised causal (2,3,3) convolution ---------------
// Work unit = 256 tokens (16x16 tile) x 128 output channels; units are dealt
// round-robin to one persistent CTA per SM (2 N-halves per tile double the
// number of units, so the tail wave is ~1/13 instead of ~1/2 of a wave).
// Roles: warp 0 lane 0 = TMA producer (halos + weight k-blocks, running ahead
// across units), warp 1 lane 0 = MMA issuer, warps 2..9 = epilogue.  The two
// M=128 accumulators of a unit take 256 TMEM columns; units alternate between
// columns 0..255 and 256..511, so the epilogue of unit i (tcgen05.ld, bias,
// SiLU, residual, bf16 stores) runs while the MMAs of unit i+1 issue.
namespace c233p {
constexpr int TILE = 16, PITCH = 18, HROWS = 18;
constexpr int HALO_BYTES = PITCH * HROWS * 128;
constexpr int HALO_STRIDE = (HALO_BYTES + 1023) / 1024 * 1024;
constexpr int BN = 128;
constexpr int B_BYTES = BN * 128;
constexpr int HSLOTS = 2, BSTAGES = 8;
constexpr int SMEM = HSLOTS * HALO_STRIDE + BSTAGES * B_BYTES + 1024 + 512;
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 64 + EPI_WARPS * 32;
}  // namespace c233p

__global__ void __launch_bounds__(c233p::THREADS, 1)
    k_lt_conv233p(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const ConvArgs a, int n_units, int n_halves) {
  using namespace c233p;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sH = smem;
  uint8_t* sB = smem + HSLOTS * HALO_STRIDE;
  uint64_t* hfull = reinterpret_cast<uint64_t*>(sB + BSTAGES * B_BYTES);
  uint64_t* hempty = hfull + HSLOTS;
  uint64_t* bfull = hempty + HSLOTS;
  uint64_t* bempty = bfull + BSTAGES;
  uint64_t* afull = bempty + BSTAGES;    // [2] accumulator ready (MMA -> epilogue)
  uint64_t* aempty = afull + 2;          // [2] accumulator drained (epilogue -> MMA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
    for (int i = 0; i < HSLOTS; ++i) { mbar_init(&hfull[i], 1); mbar_init(&hempty[i], 1); }
    for (int i = 0; i < BSTAGES; ++i) { mbar_init(&bfull[i], 1); mbar_init(&bempty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&afull[i], 1); mbar_init(&aempty[i], EPI_WARPS); }
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  const int nh = 2 * a.kb_per_tap;   // halos per unit: (temporal tap, channel block)
  const int C = a.kb_per_tap * BK;
  auto decode = [&](int u, int& g, int& t, int& x0, int& y0, int& n0) {
    int tile = u / n_halves;
    n0 = (u - tile * n_halves) * BN;
    const int tx = tile % a.tiles_x; tile /= a.tiles_x;
    const int ty = tile % a.tiles_y; tile /= a.tiles_y;
    t = a.t_lo + tile % a.t_cnt;
    g = tile / a.t_cnt;
    x0 = tx * TILE; y0 = ty * TILE;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer ----
      int hc = 0, bc = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        int g, t, x0, y0, n0;
        decode(u, g, t, x0, y0, n0);
        for (int hi = 0; hi < nh; ++hi, ++hc) {
          const int kt = hi / a.kb_per_tap, cb = hi - kt * a.kb_per_tap;
          const int hs = hc % HSLOTS;
          if (hc >= HSLOTS) mbar_wait(&hempty[hs], ((hc / HSLOTS) - 1) & 1);
          mbar_expect_tx(&hfull[hs], HALO_BYTES);
          tc::tma_load_5d(sH + hs * HALO_STRIDE, &tmA, cb * BK, x0 - 1, y0 - 1, t + kt - 1, g,
                          &hfull[hs]);
          for (int sp = 0; sp < 9; ++sp, ++bc) {
            const int bs = bc % BSTAGES;
            if (bc >= BSTAGES) mbar_wait(&bempty[bs], ((bc / BSTAGES) - 1) & 1);
            mbar_expect_tx(&bfull[bs], B_BYTES);
            tc::tma_load_2d(sB + bs * B_BYTES, &tmB, (kt * 9 + sp) * C + cb * BK, n0, &bfull[bs]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer ----
      constexpr uint32_t idesc = tc::idesc_bf16_f32(128, BN);
      int hc = 0, bc = 0, it = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++it) {
        const int ab = it & 1;
        if (it >= 2) mbar_wait(&aempty[ab], ((it >> 1) - 1) & 1);
        tc::fence_after_sync();
        const uint32_t acc = tmem + ab * 256;
        for (int hi = 0; hi < nh; ++hi, ++hc) {
          const int hs = hc % HSLOTS;
          mbar_wait(&hfull[hs], (hc / HSLOTS) & 1);
          const uint32_t hbase = smem_u32(sH + hs * HALO_STRIDE);
          for (int sp = 0; sp < 9; ++sp, ++bc) {
            const int bs = bc % BSTAGES;
            mbar_wait(&bfull[bs], (bc / BSTAGES) & 1);
            tc::fence_after_sync();
            const int dy = sp / 3, dx = sp % 3;
            const uint64_t bd = tc::smem_desc_sw128(smem_u32(sB + bs * B_BYTES));
#pragma unroll
            for (int half = 0; half < 2; ++half) {
              const uint64_t ad = halo_desc(hbase + (uint32_t)((dy * PITCH + dx + 8 * half) * 128));
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)
                tc::mma_bf16(acc + half * BN, ad + 2 * k, bd + 2 * k, idesc, (hi | sp | k) != 0);
            }
            tc::mma_commit(&bempty[bs]);
          }
          tc::mma_commit(&hempty[hs]);
        }
        tc::mma_commit(&afull[ab]);
      }
    }
  } else {
    // ---- epilogue warps: warp w drains half (w-2)/4, TMEM lanes 32*(w%4) ----
    const int e = warp - 2;
    const int half = e >> 2, q = warp & 3;
    const int m = q * 32 + lane;
    int it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++it) {
      int g, t, x0, y0, n0;
      decode(u, g, t, x0, y0, n0);
      const int ab = it & 1;
      mbar_wait(&afull[ab], (it >> 1) & 1);
      tc::fence_after_sync();
      const int y = y0 + (m >> 3), x = x0 + half * 8 + (m & 7);
      const bool valid = y < a.Ht && x < a.Wt;
      const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + ab * 256 + half * BN;
      const size_t tok = (((size_t)g * a.out_T + t) * a.Ht + y) * a.Wt + x;
      __nv_bfloat16* outp = a.out + tok * a.N + n0;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        float v[32];
        tc::tmem_ld32(trow + c, v);
        if (c + 32 == BN) {
          // last TMEM read of this accumulator by this warp: release it early
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&aempty[ab]);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          v[i] += __ldg(a.bias + n0 + c + i);
          if (a.act) v[i] = silu(v[i]);
        }
        if (!valid) continue;
        if (a.residual != nullptr) {
          const uint4* rp = reinterpret_cast<const uint4*>(a.residual + tok * a.N + n0 + c);
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            uint4 uu = __ldg(rp + qq);
            const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&uu);
#pragma unroll
            for (int e2 = 0; e2 < 4; ++e2) {
              float2 f = __bfloat1622float2(h2[e2]);
              v[qq * 8 + 2 * e2] += f.x;
              v[qq * 8 + 2 * e2 + 1] += f.y;
            }
          }
        }
        uint4* op = reinterpret_cast<uint4*>(outp + c);
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          uint4 uu;
          __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&uu);
#pragma unroll
          for (int e2 = 0; e2 < 4; ++e2)
            h2[e2] = __floats2bfloat162_rn(v[qq * 8 + 2 * e2], v[qq * 8 + 2 * e2 + 1]);
          op[qq] = uu;
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc::tmem_dealloc(tmem, 512);
  }
}

// ---- causal (2,3,3) convolution on CTA pairs (cta_group::2) ----------------
// A cluster of 2 CTAs on one TPC computes a unit of 256 tokens (16x16) x 256
// output channels with tcgen05.mma.cta_group::2 (M=256, N=256, K=16): CTA r
// owns the tokens of x-half r (its own 10x18 halo and its 128 accumulator rows)
// and loads weight rows n = 128r..128r+127 of every k-block; the MMA reads A
// and B from both CTAs' shared memory at the same offsets.  Per SM and k-step
// that is 128x256x16 of work for 4 KB of A and 4 KB of B shared-memory reads
// (the single-CTA kernel needs 8 KB for 128x128x16).  The leader's warp 1 lane
// 0 issues all MMAs; both CTAs' TMA bytes complete on the leader's barriers
// (peer bit cleared); commits multicast to both CTAs; the 8 epilogue warps of
// each CTA drain their own TMEM and arrive on the leader's accumulator-empty
// barrier through the cluster window.  Two 256-column accumulators per CTA.
namespace c233c {
constexpr int TILE = 16, PITCH = 10, HROWS = 18;
constexpr int HALO_BYTES = PITCH * HROWS * 128;                   // 23040 (1x1: 8x16 box, 16384)
constexpr int HALO_STRIDE = (HALO_BYTES + 1023) / 1024 * 1024;    // 23552
constexpr int BNH = 128;                                          // weight rows per CTA
constexpr int HSLOTS = 3, BSTAGES = 8;
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 64 + EPI_WARPS * 32;
}  // namespace c233c

__device__ __forceinline__ uint64_t halo_desc_pitch(uint32_t saddr, int pitch) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((pitch * 128) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// kHalo = true: causal (2,3,3) conv (2 temporal taps x 9 spatial taps per
// halo); false: 1x1 conv / GEMM (one tap, an 8x16 token box per CTA, temporal
// offset taps[0][0]).  A unit covers 256 output channels n_blk*256..+255.
// kTma: STORE epilogue through a swizzled smem staging tile + 5-D TMA store
// (short-K 1x1 GEMMs, whose cost is the output write); otherwise direct
// 16-byte stores from registers.
// Operand ring depths.  Halo convs: 3 halo slots (23 KB) x 8 weight stages.
// 1x1 GEMMs (a 16 KB token box per k-block, K = 4..24 k-blocks): 5 + 5
// (TMA-store epilogue, whose 64 KB staging tile takes the rest) or 5 + 8
// (pixels) -- the producer runs a whole 4-k-block unit ahead, which the
// short-K, HBM-bound GEMMs need to keep enough bytes in flight.
template <bool kHalo, bool kTma>
__host__ __device__ constexpr int pair_bstages() { return kHalo ? c233c::BSTAGES : (kTma ? 5 : 8); }
template <bool kHalo>
__host__ __device__ constexpr int pair_hslots() { return kHalo ? c233c::HSLOTS : 5; }
template <bool kHalo>
__host__ __device__ constexpr int pair_hstride() { return kHalo ? c233c::HALO_STRIDE : 16384; }
// kPix: PIXELS epilogue (unpatchify), units of 192 output channels (one frame's
// 8x8x3 patch), 96 weight rows per CTA
template <bool kPix>
__host__ __device__ constexpr int pair_bbytes() { return (kPix ? 96 : c233c::BNH) * 128; }
// epilogue staging: TMA-store tiles (kTma) or per-warp pixel rows (kPix:
// 8 warps x 4 rows x 768 B, for coalesced frame stores)
template <bool kTma, bool kPix>
__host__ __device__ constexpr int pair_stage() { return kTma ? 2 * 2 * 16384 : (kPix ? 8 * 3072 : 0); }
template <bool kHalo, bool kTma, bool kPix = false>
__host__ __device__ constexpr int pair_smem() {
  return pair_hslots<kHalo>() * pair_hstride<kHalo>() + pair_bstages<kHalo, kTma>() * pair_bbytes<kPix>() +
         pair_stage<kTma, kPix>() + 1024 + 512;
}
static_assert(pair_smem<true, false>() <= 232448, "halo conv smem");
static_assert(pair_smem<false, true>() <= 232448, "1x1 conv smem");
static_assert(pair_smem<false, false, true>() <= 232448, "pixel conv smem");

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <bool kHalo, bool kTma, bool kPix = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(c233c::THREADS, 1)
    k_lt_convpair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const __grid_constant__ CUtensorMap tmC, const ConvArgs a, int n_units,
                  int n_blocks) {
  using namespace c233c;
  constexpr int kPitch = kHalo ? PITCH : 8;
  constexpr int kBoxBytes = kHalo ? HALO_BYTES : 8 * 16 * 128;
  constexpr int kSpatial = kHalo ? 9 : 1;
  constexpr int BSTAGES = pair_bstages<kHalo, kTma>();
  constexpr int HSLOTS = pair_hslots<kHalo>();
  constexpr int HALO_STRIDE = pair_hstride<kHalo>();
  constexpr int kNU = kPix ? 192 : 256;          // output channels per unit
  constexpr int kBNH = kNU / 2;                  // weight rows per CTA
  constexpr int B_BYTES = pair_bbytes<kPix>();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sH = smem;
  uint8_t* sB = smem + HSLOTS * HALO_STRIDE;
  uint8_t* sStage = sB + BSTAGES * B_BYTES;            // kTma: [2 halves][2 boxes][128 rows][128 B]
  uint64_t* hfull = reinterpret_cast<uint64_t*>(sStage + pair_stage<kTma, kPix>());
  uint64_t* hempty = hfull + HSLOTS;
  uint64_t* bfull = hempty + HSLOTS;
  uint64_t* bempty = bfull + BSTAGES;
  uint64_t* afull = bempty + BSTAGES;
  uint64_t* aempty = afull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_ctarank();
  const bool leader = rank == 0;
  if (threadIdx.x == 0) {
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
    if (kTma) tc::prefetch_tmap(&tmC);
    for (int i = 0; i < HSLOTS; ++i) { mbar_init(&hfull[i], 1); mbar_init(&hempty[i], 1); }
    for (int i = 0; i < BSTAGES; ++i) { mbar_init(&bfull[i], 1); mbar_init(&bempty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&afull[i], 1); mbar_init(&aempty[i], 2 * EPI_WARPS); }
    fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc_pair(tmem_slot, 512);
  tc::fence_before_sync();
  tc::cluster_sync();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  const int nh = (kHalo ? 2 : 1) * a.kb_per_tap;
  const int C = a.kb_per_tap * BK;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  auto decode = [&](int u, int& g, int& t, int& x0, int& y0, int& nb) {
    int tile = u / n_blocks;
    nb = u - tile * n_blocks;
    const int tx = tile % a.tiles_x; tile /= a.tiles_x;
    const int ty = tile % a.tiles_y; tile /= a.tiles_y;
    t = a.t_lo + tile % a.t_cnt;
    g = tile / a.t_cnt;
    x0 = tx * TILE; y0 = ty * TILE;
  };
  // at t = 0 the causal conv's temporal tap t-1 reads only zero padding:
  // skip its halo loads and MMAs (the same sums: the skipped products are 0)
  auto first_hi = [&](int t) { return (kHalo && t == 0) ? a.kb_per_tap : 0; };

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer (both CTAs): own halo, own half of the weights ----
      int hc = 0, bc = 0;
      for (int u = pair; u < n_units; u += npairs) {
        int g, t, x0, y0, nb;
        decode(u, g, t, x0, y0, nb);
        for (int hi = first_hi(t); hi < nh; ++hi, ++hc) {
          const int kt = hi / a.kb_per_tap, cb = hi - kt * a.kb_per_tap;
          const int hs = hc % HSLOTS;
          if (hc >= HSLOTS) mbar_wait(&hempty[hs], ((hc / HSLOTS) - 1) & 1);
          if (leader) mbar_expect_tx(&hfull[hs], 2 * kBoxBytes);
          if (kHalo)
            tc::tma_load_5d_pair(sH + hs * HALO_STRIDE, &tmA, cb * BK, x0 + 8 * (int)rank - 1,
                                 y0 - 1, t + kt - 1, g, &hfull[hs]);
          else
            tc::tma_load_5d_pair(sH + hs * HALO_STRIDE, &tmA, cb * BK, x0 + 8 * (int)rank, y0,
                                 t + a.taps[0][0], g, &hfull[hs]);
          for (int sp = 0; sp < kSpatial; ++sp, ++bc) {
            const int bs = bc % BSTAGES;
            if (bc >= BSTAGES) mbar_wait(&bempty[bs], ((bc / BSTAGES) - 1) & 1);
            if (leader) mbar_expect_tx(&bfull[bs], 2 * B_BYTES);
            tc::tma_load_2d_pair(sB + bs * B_BYTES, &tmB, (kt * kSpatial + sp) * C + cb * BK,
                                 nb * kNU + (int)rank * kBNH, &bfull[bs]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---- MMA issuer (leader only): M=256 across the pair, N=256 ----
      constexpr uint32_t idesc = tc::idesc_bf16_f32(256, kNU);
      int hc = 0, bc = 0, it = 0;
      for (int u = pair; u < n_units; u += npairs, ++it) {
        int g, t, x0, y0, nb;
        decode(u, g, t, x0, y0, nb);
        const int hi0 = first_hi(t);
        const int ab = it & 1;
        if (it >= 2) mbar_wait(&aempty[ab], ((it >> 1) - 1) & 1);
        tc::fence_after_sync();
        const uint32_t acc = tmem + ab * 256;
        for (int hi = hi0; hi < nh; ++hi, ++hc) {
          const int hs = hc % HSLOTS;
          mbar_wait(&hfull[hs], (hc / HSLOTS) & 1);
          const uint32_t hbase = smem_u32(sH + hs * HALO_STRIDE);
          for (int sp = 0; sp < kSpatial; ++sp, ++bc) {
            const int bs = bc % BSTAGES;
            mbar_wait(&bfull[bs], (bc / BSTAGES) & 1);
            tc::fence_after_sync();
            const int dy = sp / 3, dx = sp % 3;
            const uint64_t bd = tc::smem_desc_sw128(smem_u32(sB + bs * B_BYTES));
            const uint64_t ad = halo_desc_pitch(hbase + (uint32_t)((dy * kPitch + dx) * 128), kPitch);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              tc::mma_bf16_pair(acc, ad + 2 * k, bd + 2 * k, idesc, (hi != hi0 || sp | k) != 0);
            tc::mma_commit_pair(&bempty[bs]);
          }
          tc::mma_commit_pair(&hempty[hs]);
        }
        tc::mma_commit_pair(&afull[ab]);
      }
    }
  } else {
    // ---- epilogue (both CTAs): warp w drains columns 128*((w-2)/4).., lanes 32*(w%4) ----
    const int e = warp - 2;
    const int half = e >> 2, q = warp & 3;
    const int m = q * 32 + lane;
    const uint32_t aempty_leader = tc::mapa(smem_u32(&aempty[0]), 0);
    const bool issuer = kTma && (e & 3) == 0 && lane == 0;     // first warp of each half
    int it = 0;
    for (int u = pair; u < n_units; u += npairs, ++it) {
      int g, t, x0, y0, nb;
      decode(u, g, t, x0, y0, nb);
      const int ab = it & 1;
      mbar_wait(&afull[ab], (it >> 1) & 1);
      tc::fence_after_sync();
      const int y = y0 + (m >> 3), x = x0 + 8 * (int)rank + (m & 7);
      const bool valid = y < a.Ht && x < a.Wt;
      if (kPix) {
        // ---- unpatchify: columns half*96 .. +95 = pixel rows py = 4*half .. +3 of frame f ----
        const uint32_t trp = tmem + ((uint32_t)(q * 32) << 16) + ab * 256 + half * 96;
        float v[96];
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
          float u32[32];
          tc::tmem_ld32(trp + cc * 32, u32);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[cc * 32 + i] = u32[i];
        }
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_cluster_relaxed(aempty_leader + ab * 8);
        const int f = a.frame_base + nb;
        const int nb0 = nb * kNU + half * 96;
        const float4* bp4 = reinterpret_cast<const float4*>(a.bias + nb0);
#pragma unroll
        for (int i4 = 0; i4 < 24; ++i4) {
          const float4 bb = __ldg(bp4 + i4);
          v[4 * i4 + 0] = fminf(fmaxf(v[4 * i4 + 0] + bb.x, 0.0f), 1.0f);
          v[4 * i4 + 1] = fminf(fmaxf(v[4 * i4 + 1] + bb.y, 0.0f), 1.0f);
          v[4 * i4 + 2] = fminf(fmaxf(v[4 * i4 + 2] + bb.z, 0.0f), 1.0f);
          v[4 * i4 + 3] = fminf(fmaxf(v[4 * i4 + 3] + bb.w, 0.0f), 1.0f);
        }
        const bool vec = (a.w & 3) == 0;
        // warp = 4 token rows x the pair-half's 8 tokens: each pixel row of it
        // is 8 x 8 px x 3 = 192 contiguous floats when all 8 tokens are inside
        const int xs = x0 + 8 * (int)rank;                 // first token of the warp's rows
        const bool seg = vec && xs + 8 <= a.Wt && xs * 8 + 64 <= a.w;
        if (seg) {
          float* srow = reinterpret_cast<float*>(sStage) + (warp - 2) * 768;   // [4][192]
#pragma unroll
          for (int pr = 0; pr < 4; ++pr) {
            float4* s4 = reinterpret_cast<float4*>(srow + (lane >> 3) * 192 + (lane & 7) * 24);
#pragma unroll
            for (int e4 = 0; e4 < 6; ++e4)
              s4[e4] = make_float4(v[pr * 24 + 4 * e4], v[pr * 24 + 4 * e4 + 1],
                                   v[pr * 24 + 4 * e4 + 2], v[pr * 24 + 4 * e4 + 3]);
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 6; ++i) {
              const int idx = i * 32 + lane, r = idx / 48, c4 = idx - r * 48;
              const int yr = y0 + q * 4 + r;                 // token row of staged row r
              const int Y = yr * 8 + half * 4 + pr;
              if (yr < a.Ht && Y < a.h) {
                float4* d4 = reinterpret_cast<float4*>(
                    a.frames + ((((size_t)g * 9 + f) * a.h + Y) * a.w + xs * 8) * 3);
                d4[c4] = reinterpret_cast<const float4*>(srow + r * 192)[c4];
              }
            }
            __syncwarp();
          }
          continue;
        }
        if (!valid) continue;
#pragma unroll
        for (int pr = 0; pr < 4; ++pr) {
          const int Y = y * 8 + half * 4 + pr;
          if (Y >= a.h) continue;
          const int X0 = x * 8;
          float* dst = a.frames + ((((size_t)g * 9 + f) * a.h + Y) * a.w + X0) * 3;
          if (vec && X0 + 8 <= a.w) {
            float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
            for (int e4 = 0; e4 < 6; ++e4)
              d4[e4] = make_float4(v[pr * 24 + 4 * e4], v[pr * 24 + 4 * e4 + 1],
                                   v[pr * 24 + 4 * e4 + 2], v[pr * 24 + 4 * e4 + 3]);
          } else {
            const int npx = min(8, a.w - X0);
#pragma unroll
            for (int e4 = 0; e4 < 24; ++e4)
              if (e4 / 3 < npx) dst[e4] = v[pr * 24 + e4];
          }
        }
        continue;
      }
      const int n0 = nb * 256 + half * 128;
      const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + ab * 256 + half * 128;
      const size_t tok = (((size_t)g * a.out_T + t) * a.Ht + y) * a.Wt + x;
      __nv_bfloat16* outp = a.out + tok * a.N + n0;
      if constexpr (kTma) {
        // ---- short-K GEMM epilogue (HBM-bound): this row's 128 residual
        // values are fetched up front (one memory latency per unit, not one
        // per 32-column chunk), and the wait for the previous unit's TMA
        // store to release the staging tile is deferred to the first
        // staging write, so it overlaps the TMEM drain and the loads ----
        uint8_t* stage = sStage + half * 2 * 16384;
        uint4 res[16];
        const bool has_res = valid && a.residual != nullptr;
        if (has_res) {
          const uint4* rp = reinterpret_cast<const uint4*>(a.residual + tok * a.N + n0);
#pragma unroll
          for (int i = 0; i < 16; ++i) res[i] = __ldg(rp + i);
        }
#pragma unroll
        for (int c = 0; c < 128; c += 32) {
          float v[32];
          tc::tmem_ld32(trow + c, v);
          if (c + 32 == 128) {
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive_cluster_relaxed(aempty_leader + ab * 8);
          }
          const float4* bp = reinterpret_cast<const float4*>(a.bias + n0 + c);
#pragma unroll
          for (int i4 = 0; i4 < 8; ++i4) {
            const float4 bb = __ldg(bp + i4);
            v[4 * i4 + 0] += bb.x;
            v[4 * i4 + 1] += bb.y;
            v[4 * i4 + 2] += bb.z;
            v[4 * i4 + 3] += bb.w;
          }
          if (a.act) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = silu(v[i]);
          }
          if (has_res) {
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
              const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&res[(c >> 3) + qq]);
#pragma unroll
              for (int e2 = 0; e2 < 4; ++e2) {
                float2 f = __bfloat1622float2(h2[e2]);
                v[qq * 8 + 2 * e2] += f.x;
                v[qq * 8 + 2 * e2 + 1] += f.y;
              }
            }
          }
          if (c == 0) {
            // the previous unit's TMA store has read the staging tile
            if (issuer) tma_store_wait_read();
            named_bar(1 + half, 128);
          }
          const int box = c >> 6, j0 = (c & 63) >> 3;
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            uint4 uu;
            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&uu);
#pragma unroll
            for (int e2 = 0; e2 < 4; ++e2)
              h2[e2] = __floats2bfloat162_rn(v[qq * 8 + 2 * e2], v[qq * 8 + 2 * e2 + 1]);
            const int j = j0 + qq;
            *reinterpret_cast<uint4*>(stage + box * 16384 + m * 128 + ((j ^ (m & 7)) << 4)) = uu;
          }
        }
        fence_proxy_async_smem();
        named_bar(1 + half, 128);
        if (issuer) {
#pragma unroll
          for (int b = 0; b < 2; ++b)
            tc::tma_store_5d(&tmC, stage + b * 16384, n0 + b * 64, x0 + 8 * (int)rank, y0, t, g);
          tma_store_commit();
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < 128; c += 32) {
          float v[32];
          tc::tmem_ld32(trow + c, v);
          if (c + 32 == 128) {
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive_cluster_relaxed(aempty_leader + ab * 8);
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            v[i] += __ldg(a.bias + n0 + c + i);
            if (a.act) v[i] = silu(v[i]);
          }
          if (!valid) continue;
          if (a.residual != nullptr) {
            const uint4* rp = reinterpret_cast<const uint4*>(a.residual + tok * a.N + n0 + c);
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
              uint4 uu = __ldg(rp + qq);
              const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&uu);
#pragma unroll
              for (int e2 = 0; e2 < 4; ++e2) {
                float2 f = __bfloat1622float2(h2[e2]);
                v[qq * 8 + 2 * e2] += f.x;
                v[qq * 8 + 2 * e2 + 1] += f.y;
              }
            }
          }
          uint4* op = reinterpret_cast<uint4*>(outp + c);
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            uint4 uu;
            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&uu);
#pragma unroll
            for (int e2 = 0; e2 < 4; ++e2)
              h2[e2] = __floats2bfloat162_rn(v[qq * 8 + 2 * e2], v[qq * 8 + 2 * e2 + 1]);
            op[qq] = uu;
          }
        }
      }
    }
    if (issuer) tma_store_wait_all();
  }
  tc::fence_before_sync();
  tc::cluster_sync();
  if (warp == 1) {
    __syncwarp();
    tc::tmem_dealloc_pair(tmem, 512);
  }
}

// ---- causal spatio-temporal window attention (the attention core) ---------
// Q, K, V come from one tcgen05 1x1 projection (qkv [G][2][H'][W'][3D], channel
// = part*D + head*64 + d).  A CTA owns one 8x8 token window of one GoP and one
// 64-dim head: 128 threads = 2 latent frames x 64 query tokens.  Keys/values of
// the window's two frames are staged in shared memory as fp32; a query of frame
// t attends to the window's valid tokens of frames <= t (causal in time), with
// a one-pass online softmax in fp32.  The core is ~0.5 % of the tokenizer's
// flops (64-128 keys per query), so it is plain SIMT; the projections around
// it are the tensor-core GEMMs.
constexpr int ATT_WIN = 8, ATT_HD = 64;

__global__ void __launch_bounds__(128)
    k_lt_attn(const __nv_bfloat16* __restrict__ qkv, int G, int Ht, int Wt, int D,
              __nv_bfloat16* __restrict__ out) {
  extern __shared__ float4 att_smem[];      // K [128][16], V [128][16] float4, kval[128]
  float4 (*Ks)[ATT_HD / 4] = reinterpret_cast<float4 (*)[ATT_HD / 4]>(att_smem);
  float4 (*Vs)[ATT_HD / 4] = reinterpret_cast<float4 (*)[ATT_HD / 4]>(att_smem + 128 * (ATT_HD / 4));
  int* kval = reinterpret_cast<int*>(att_smem + 2 * 128 * (ATT_HD / 4));
  const int wins_x = ceil_div(Wt, ATT_WIN);
  const int wy = blockIdx.x / wins_x, wx = blockIdx.x - wy * wins_x;
  const int head = blockIdx.y, g = blockIdx.z;
  const int t = threadIdx.x;
  const int ft = t >> 6, lt = t & 63;
  const int y = wy * ATT_WIN + (lt >> 3), x = wx * ATT_WIN + (lt & 7);
  const bool valid = y < Ht && x < Wt;
  const size_t tok = (((size_t)g * 2 + ft) * Ht + y) * Wt + x;
  const int C3 = 3 * D;
  // stage this thread's key / value row (token t of the window) as fp32
  kval[t] = valid;
  {
    float4* kd = Ks[t];
    float4* vd = Vs[t];
    if (valid) {
      const uint4* kp = reinterpret_cast<const uint4*>(qkv + tok * C3 + D + head * ATT_HD);
      const uint4* vp = reinterpret_cast<const uint4*>(qkv + tok * C3 + 2 * D + head * ATT_HD);
#pragma unroll
      for (int i = 0; i < ATT_HD / 8; ++i) {
        uint4 ku = __ldg(kp + i), vu = __ldg(vp + i);
        const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&ku);
        const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&vu);
        float2 a0 = __bfloat1622float2(k2[0]), a1 = __bfloat1622float2(k2[1]);
        float2 a2 = __bfloat1622float2(k2[2]), a3 = __bfloat1622float2(k2[3]);
        kd[2 * i] = make_float4(a0.x, a0.y, a1.x, a1.y);
        kd[2 * i + 1] = make_float4(a2.x, a2.y, a3.x, a3.y);
        a0 = __bfloat1622float2(v2[0]); a1 = __bfloat1622float2(v2[1]);
        a2 = __bfloat1622float2(v2[2]); a3 = __bfloat1622float2(v2[3]);
        vd[2 * i] = make_float4(a0.x, a0.y, a1.x, a1.y);
        vd[2 * i + 1] = make_float4(a2.x, a2.y, a3.x, a3.y);
      }
    }
  }
  float q[ATT_HD];
  if (valid) {
    const uint4* qp = reinterpret_cast<const uint4*>(qkv + tok * C3 + head * ATT_HD);
#pragma unroll
    for (int i = 0; i < ATT_HD / 8; ++i) {
      uint4 u = __ldg(qp + i);
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 f = __bfloat1622float2(h2[e]);
        q[8 * i + 2 * e] = f.x * 0.125f;          // 1/sqrt(64), exact
        q[8 * i + 2 * e + 1] = f.y * 0.125f;
      }
    }
  }
  __syncthreads();
  if (!valid) return;
  float acc[ATT_HD];
#pragma unroll
  for (int d = 0; d < ATT_HD; ++d) acc[d] = 0.0f;
  float m = -INFINITY, l = 0.0f;
  const int nkeys = (ft + 1) * ATT_WIN * ATT_WIN;   // causal: frames 0..ft
  for (int j = 0; j < nkeys; ++j) {
    if (!kval[j]) continue;
    float sdot = 0.0f;
#pragma unroll
    for (int i = 0; i < ATT_HD / 4; ++i) {
      const float4 k4 = Ks[j][i];
      sdot = fmaf(q[4 * i], k4.x, sdot);
      sdot = fmaf(q[4 * i + 1], k4.y, sdot);
      sdot = fmaf(q[4 * i + 2], k4.z, sdot);
      sdot = fmaf(q[4 * i + 3], k4.w, sdot);
    }
    const float mn = fmaxf(m, sdot);
    const float c = __expf(m - mn), p = __expf(sdot - mn);
    l = l * c + p;
#pragma unroll
    for (int i = 0; i < ATT_HD / 4; ++i) {
      const float4 v4 = Vs[j][i];
      acc[4 * i] = fmaf(p, v4.x, acc[4 * i] * c);
      acc[4 * i + 1] = fmaf(p, v4.y, acc[4 * i + 1] * c);
      acc[4 * i + 2] = fmaf(p, v4.z, acc[4 * i + 2] * c);
      acc[4 * i + 3] = fmaf(p, v4.w, acc[4 * i + 3] * c);
    }
    m = mn;
  }
  const float inv = 1.0f / l;
  uint4* op = reinterpret_cast<uint4*>(out + tok * D + head * ATT_HD);
#pragma unroll
  for (int i = 0; i < ATT_HD / 8; ++i) {
    uint4 u;
    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      h2[e] = __floats2bfloat162_rn(acc[8 * i + 2 * e] * inv, acc[8 * i + 2 * e + 1] * inv);
    op[i] = u;
  }
}

// ---- causal window attention core on tcgen05 --------------------------------
// One CTA = one (GoP, 8x8 window, 64-dim head): 128 query rows (2 latent
// frames x 64 tokens) and the same 128 keys.  Q, K and V^T are staged into
// 128B-swizzled K-major tiles with st.shared (manual swizzle), then
//   S = Q K^T   tcgen05.mma M=128 N=128 K=64  -> TMEM columns 0..127
//   softmax     thread q: tcgen05.ld its 128 scores, causal + validity mask,
//               P = exp((s - max) / 8) rounded to bf16 -> smem (over Q, K)
//   O = P V     tcgen05.mma M=128 N=64 K=128  -> TMEM columns 0..63
//   O / l       tcgen05.ld, bf16 stores.
constexpr int ATT_SMEM = 3 * 16384 + 1024 + 64 + 128 * 4;

__global__ void __launch_bounds__(128)
    k_lt_attn_tc(const __nv_bfloat16* __restrict__ qkv, int G, int Ht, int Wt, int D,
                 __nv_bfloat16* __restrict__ out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;                 // [128 q][64 d]   A of S
  uint8_t* sK = smem + 16384;         // [128 k][64 d]   B of S
  uint8_t* sP = smem;                 // [2 kb][128 q][64 k] A of O (reuses sQ, sK)
  uint8_t* sV = smem + 32768;         // [2 kb][64 d][64 k]  B of O (V^T)
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 49152);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2);
  int* kval = reinterpret_cast<int*>(smem + 49152 + 64);

  const int wins_x = ceil_div(Wt, ATT_WIN);
  const int wy = blockIdx.x / wins_x, wx = blockIdx.x - wy * wins_x;
  const int head = blockIdx.y, g = blockIdx.z;
  const int t = threadIdx.x, warp = t >> 5;
  const int ft = t >> 6, lt = t & 63;
  const int y = wy * ATT_WIN + (lt >> 3), x = wx * ATT_WIN + (lt & 7);
  const bool valid = y < Ht && x < Wt;
  const size_t tok = (((size_t)g * 2 + ft) * Ht + y) * Wt + x;
  const int C3 = 3 * D;

  if (t == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 128);

  // ---- stage Q, K rows (K-major, row = token t) and V^T (row = dim) ----
  kval[t] = valid;
  {
    uint4 q4[8], k4[8], v4[8];
    if (valid) {
      const uint4* base = reinterpret_cast<const uint4*>(qkv + tok * C3 + head * ATT_HD);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        q4[j] = __ldg(base + j);
        k4[j] = __ldg(base + D / 8 + j);
        v4[j] = __ldg(base + 2 * D / 8 + j);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) q4[j] = k4[j] = v4[j] = make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int off = t * 128 + ((j ^ (t & 7)) << 4);
      *reinterpret_cast<uint4*>(sQ + off) = q4[j];
      *reinterpret_cast<uint4*>(sK + off) = k4[j];
    }
    const int kb = t >> 6, kk = t & 63;
    uint8_t* vb = sV + kb * 8192 + (kk & 7) * 2;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v4[j]);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int d = 8 * j + i;
        *reinterpret_cast<__nv_bfloat16*>(vb + d * 128 + (((kk >> 3) ^ (d & 7)) << 4)) = e[i];
      }
    }
  }
  fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (t == 0) {
    constexpr uint32_t id1 = tc::idesc_bf16_f32(128, 128);
    const uint64_t ad = tc::smem_desc_sw128(smem_u32(sQ));
    const uint64_t bd = tc::smem_desc_sw128(smem_u32(sK));
#pragma unroll
    for (int k = 0; k < 4; ++k) tc::mma_bf16(tmem, ad + 2 * k, bd + 2 * k, id1, k);
    tc::mma_commit(&bar[0]);
  }
  mbar_wait(&bar[0], 0);
  tc::fence_after_sync();

  // ---- softmax of this thread's query row (TMEM lane t) ----
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  float sc[128];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    float v[32];
    tc::tmem_ld32(trow + c * 32, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) sc[c * 32 + i] = v[i];
  }
  const int nk = (ft + 1) * 64;       // causal: keys of frames <= ft
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < 128; ++k)
    if (k < nk && kval[k]) m = fmaxf(m, sc[k]);
  float l = 0.0f;
#pragma unroll
  for (int k = 0; k < 128; ++k) {
    const float p = (k < nk && kval[k]) ? __expf((sc[k] - m) * 0.125f) : 0.0f;
    sc[k] = p;
    l += p;
  }
  tc::fence_before_sync();
  __syncthreads();                    // every S read done and GEMM 1 retired: sQ/sK -> sP
#pragma unroll
  for (int kb = 0; kb < 2; ++kb) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint4 u;
      __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        h2[e] = __floats2bfloat162_rn(sc[kb * 64 + 8 * j + 2 * e], sc[kb * 64 + 8 * j + 2 * e + 1]);
      *reinterpret_cast<uint4*>(sP + kb * 16384 + t * 128 + ((j ^ (t & 7)) << 4)) = u;
    }
  }
  fence_proxy_async_smem();
  __syncthreads();
  tc::fence_after_sync();
  if (t == 0) {
    constexpr uint32_t id2 = tc::idesc_bf16_f32(128, 64);
#pragma unroll
    for (int kb = 0; kb < 2; ++kb) {
      const uint64_t ad = tc::smem_desc_sw128(smem_u32(sP + kb * 16384));
      const uint64_t bd = tc::smem_desc_sw128(smem_u32(sV + kb * 8192));
#pragma unroll
      for (int k = 0; k < 4; ++k) tc::mma_bf16(tmem, ad + 2 * k, bd + 2 * k, id2, kb | k);
    }
    tc::mma_commit(&bar[1]);
  }
  mbar_wait(&bar[1], 0);
  tc::fence_after_sync();
  float o[64];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float v[32];
    tc::tmem_ld32(trow + c * 32, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) o[c * 32 + i] = v[i];
  }
  if (valid) {
    const float inv = 1.0f / l;
    uint4* op = reinterpret_cast<uint4*>(out + tok * D + head * ATT_HD);
#pragma unroll
    for (int i = 0; i < ATT_HD / 8; ++i) {
      uint4 u;
      __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        h2[e] = __floats2bfloat162_rn(o[8 * i + 2 * e] * inv, o[8 * i + 2 * e + 1] * inv);
      op[i] = u;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 128);
}

// ---- attention epilogue helpers (k_lt_attn_fused, k_lt_attn_persist) -----
// Thread = TMEM lane = token row q of the window (q = frame * 64 + 8y + x).

// qkv accumulator row (192 TMEM columns at tq) + bias -> bf16 Q, K and V rows
// into their 128B-swizzled tiles.
__device__ __forceinline__ void att_qkv_epilogue(uint32_t tq, const float* __restrict__ bqkv, int D,
                                                 int head, bool valid, int q, uint8_t* sQ,
                                                 uint8_t* sK, uint8_t* sV) {
#pragma unroll 1
  for (int c = 0; c < 6; ++c) {
    float v[32];
    tc::tmem_ld32(tq + c * 32, v);
    const int part = c >> 1;                       // 0 q, 1 k, 2 v
    const int d0 = (c & 1) * 32;
    const float4* bp = reinterpret_cast<const float4*>(bqkv + part * D + head * ATT_HD + d0);
#pragma unroll
    for (int e4 = 0; e4 < 8; ++e4) {
      const float4 bb = __ldg(bp + e4);
      v[4 * e4 + 0] += bb.x;
      v[4 * e4 + 1] += bb.y;
      v[4 * e4 + 2] += bb.z;
      v[4 * e4 + 3] += bb.w;
    }
    if (!valid) {
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] = 0.0f;
    }
    // Q, K: K-major A / B of S = Q K^T; V: MN-major B of O = P V (row =
    // key, d contiguous) -- all three are plain swizzled 128-byte rows
    uint8_t* base = part == 0 ? sQ : (part == 1 ? sK : sV);
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      uint4 w4;
      __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&w4);
#pragma unroll
      for (int e = 0; e < 4; ++e) h2[e] = __floats2bfloat162_rn(v[qq * 8 + 2 * e], v[qq * 8 + 2 * e + 1]);
      const int j = (d0 >> 3) + qq;
      *reinterpret_cast<uint4*>(base + q * 128 + ((j ^ (q & 7)) << 4)) = w4;
    }
  }
}

// O = P V: A = P (K-major, two 64-key tiles at sP), B = V (MN-major [128
// keys][64 d] at sV); 8 MMAs of K = 16 keys.
__device__ __forceinline__ void att_issue_pv(uint32_t tmem_o, uint8_t* sP, uint8_t* sV) {
  constexpr uint32_t id2 = tc::idesc_bf16_f32_bmn(128, 64);
#pragma unroll
  for (int kb = 0; kb < 2; ++kb) {
    const uint64_t ad = tc::smem_desc_sw128(smem_u32(sP + kb * 16384));
    const uint64_t bd = tc::smem_desc_sw128(smem_u32(sV + kb * 8192));
#pragma unroll
    for (int k = 0; k < 4; ++k) tc::mma_bf16(tmem_o, ad + 2 * k, bd + 128 * k, id2, kb | k);
  }
}

// Causal window softmax of query row q from its 128 scores in TMEM (tS), two
// passes of 32 columns (row max; then exp, sum, bf16 P into the two
// 128B-swizzled K-major tiles at sP).  Key k is valid when k < 64 * (frame
// of q + 1) and its (y, x) is inside the frame (vrow / vcol: the window's
// valid rows / columns as bit masks).  p = 2^((s - m) * log2(e) / 8) with
// one FFMA + ex2.approx; keys of the later frame are skipped for frame-0
// queries (the sum order stays k = 0..127: skipped terms are +0).
// Returns the row sum l.
__device__ __forceinline__ float att_softmax_p(uint32_t tS, uint8_t* sP, int q, uint32_t vrow,
                                               uint32_t vcol) {
  constexpr float kC = 0.125f * 1.4426950408889634f;
  const int nch = ((q >> 6) + 1) * 2;              // 32-key chunks in the causal range
  const bool interior = vrow == 0xffu && vcol == 0xffu;
  float m = -INFINITY;
#pragma unroll 1
  for (int c = 0; c < nch; ++c) {
    float v[32];
    tc::tmem_ld32(tS + c * 32, v);
    if (interior) {
#pragma unroll
      for (int e = 0; e < 32; ++e) m = fmaxf(m, v[e]);
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const int kl = (c * 32 + e) & 63;
        if ((vrow >> (kl >> 3)) & (vcol >> (kl & 7)) & 1u) m = fmaxf(m, v[e]);
      }
    }
  }
  const float mc = m * kC;
  float l = 0.0f;
#pragma unroll 1
  for (int c = 0; c < 4; ++c) {
    float v[32];
    if (c < nch) {
      tc::tmem_ld32(tS + c * 32, v);
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const int kl = (c * 32 + e) & 63;
        const bool ok = interior || ((vrow >> (kl >> 3)) & (vcol >> (kl & 7)) & 1u);
        float y;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(fmaf(v[e], kC, -mc)));
        v[e] = ok ? y : 0.0f;
        l += v[e];
      }
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] = 0.0f;
    }
    uint8_t* pb = sP + (c >> 1) * 16384 + q * 128;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      uint4 w4;
      __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&w4);
#pragma unroll
      for (int e = 0; e < 4; ++e) h2[e] = __floats2bfloat162_rn(v[8 * jj + 2 * e], v[8 * jj + 2 * e + 1]);
      const int jc = (c & 1) * 4 + jj;
      *reinterpret_cast<uint4*>(pb + ((jc ^ (q & 7)) << 4)) = w4;
    }
  }
  return l;
}

// O row (64 TMEM columns at tO) / l -> bf16 output row.  Called by every
// thread of the warp (tcgen05.ld is warp-collective); only valid rows store.
__device__ __forceinline__ void att_store_o(uint32_t tO, float l, bool valid, __nv_bfloat16* orow) {
  float ov[64];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float v[32];
    tc::tmem_ld32(tO + c * 32, v);
#pragma unroll
    for (int e = 0; e < 32; ++e) ov[c * 32 + e] = v[e];
  }
  if (!valid) return;
  const float inv = 1.0f / l;
  uint4* op = reinterpret_cast<uint4*>(orow);
#pragma unroll
  for (int j = 0; j < ATT_HD / 8; ++j) {
    uint4 w4;
    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&w4);
#pragma unroll
    for (int e = 0; e < 4; ++e) h2[e] = __floats2bfloat162_rn(ov[8 * j + 2 * e] * inv, ov[8 * j + 2 * e + 1] * inv);
    op[j] = w4;
  }
}

// ---- fused qkv projection + causal window attention (tcgen05) -------------
// One CTA = (GoP, 8x8 window, 64-dim head).  The qkv projection of the
// window's 128 tokens for this head is a third tcgen05 GEMM inside the CTA:
//   QKV = H W_h^T   M=128 (2 frames x 64 tokens), N=192 (q|k|v), K=D,
// A = the window's tokens of the residual stream (two 5-D TMA boxes per
// 64-channel block, zero-filled outside the frame), B = the head's 192 rows of
// W_qkv, through a 2-stage TMA ring; the epilogue (+bias, bf16) writes Q, K
// and V straight into the swizzled operand tiles of S = QK^T and O = PV, then the
// softmax / P V steps of k_lt_attn_tc follow.  The qkv tensor never exists.
constexpr int AF_STAGE = 16384 + 24576;                 // A (128 x 64) + B (192 x 64) bf16
constexpr int AF_SMEM = 2 * AF_STAGE + 1024 + 128 + 128 * 4;

__global__ void __launch_bounds__(128)
    k_lt_attn_fused(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmW,
                    const float* __restrict__ bqkv, int G, int Ht, int Wt, int D,
                    __nv_bfloat16* __restrict__ out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;                 // after the projection: [128 q][64 d]
  uint8_t* sK = smem + 16384;         // [128 k][64 d]
  uint8_t* sP = smem;                 // [2 kb][128 q][64 k]
  uint8_t* sV = smem + 32768;         // [128 k][64 d]  (MN-major B of O = P V)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * AF_STAGE);
  uint64_t* empty = full + 2;
  uint64_t* bar = empty + 2;          // [0] qkv, [1] S, [2] O
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 3);

  const int wins_x = ceil_div(Wt, ATT_WIN);
  const int wy = blockIdx.x / wins_x, wx = blockIdx.x - wy * wins_x;
  const int head = blockIdx.y, g = blockIdx.z;
  const int t = threadIdx.x, warp = t >> 5;
  const int ft = t >> 6, lt = t & 63;
  const int y = wy * ATT_WIN + (lt >> 3), x = wx * ATT_WIN + (lt & 7);
  const bool valid = y < Ht && x < Wt;
  const size_t tok = (((size_t)g * 2 + ft) * Ht + y) * Wt + x;
  const int ncb = D / BK;

  if (t == 0) {
    tc::prefetch_tmap(&tmH);
    tc::prefetch_tmap(&tmW);
    for (int i = 0; i < 2; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 3; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 256);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  // ---- QKV projection (thread 0 streams the operands and issues the MMAs) ----
  if (t == 0) {
    auto load = [&](int cb, int s) {
      uint8_t* st = smem + s * AF_STAGE;
      mbar_expect_tx(&full[s], AF_STAGE);
      tc::tma_load_5d(st, &tmH, cb * BK, wx * ATT_WIN, wy * ATT_WIN, 0, g, &full[s]);
      tc::tma_load_5d(st + 8192, &tmH, cb * BK, wx * ATT_WIN, wy * ATT_WIN, 1, g, &full[s]);
      for (int part = 0; part < 3; ++part)
        tc::tma_load_2d(st + 16384 + part * 8192, &tmW, cb * BK, part * D + head * ATT_HD, &full[s]);
    };
    for (int cb = 0; cb < ncb && cb < 2; ++cb) load(cb, cb);
    constexpr uint32_t id0 = tc::idesc_bf16_f32(128, 192);
    for (int cb = 0; cb < ncb; ++cb) {
      const int s = cb & 1;
      mbar_wait(&full[s], (cb >> 1) & 1);
      tc::fence_after_sync();
      const uint64_t ad = tc::smem_desc_sw128(smem_u32(smem + s * AF_STAGE));
      const uint64_t bd = tc::smem_desc_sw128(smem_u32(smem + s * AF_STAGE + 16384));
#pragma unroll
      for (int k = 0; k < BK / 16; ++k) tc::mma_bf16(tmem, ad + 2 * k, bd + 2 * k, id0, cb | k);
      tc::mma_commit(&empty[s]);
      if (cb + 2 < ncb) {
        mbar_wait(&empty[s], (cb >> 1) & 1);
        load(cb + 2, s);
      }
    }
    tc::mma_commit(&bar[0]);
  }
  mbar_wait(&bar[0], 0);
  tc::fence_after_sync();

  // ---- +bias, bf16: Q, K and V rows into their tiles ----
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  att_qkv_epilogue(trow, bqkv, D, head, valid, t, sQ, sK, sV);
  fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();

  if (t == 0) {
    constexpr uint32_t id1 = tc::idesc_bf16_f32(128, 128);
    const uint64_t ad = tc::smem_desc_sw128(smem_u32(sQ));
    const uint64_t bd = tc::smem_desc_sw128(smem_u32(sK));
#pragma unroll
    for (int k = 0; k < 4; ++k) tc::mma_bf16(tmem, ad + 2 * k, bd + 2 * k, id1, k);
    tc::mma_commit(&bar[1]);
  }
  mbar_wait(&bar[1], 0);
  tc::fence_after_sync();
  const uint32_t vrow = (1u << min(8, Ht - wy * ATT_WIN)) - 1u;
  const uint32_t vcol = (1u << min(8, Wt - wx * ATT_WIN)) - 1u;
  // P overwrites Q and K: every thread's S reads and GEMM 1 (s barrier) are
  // done before any P store -- the S GEMM completed (bar[1]) and P rows are
  // per-thread, while S lives in TMEM
  const float l = att_softmax_p(trow, sP, t, vrow, vcol);
  fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (t == 0) {
    att_issue_pv(tmem, sP, sV);
    tc::mma_commit(&bar[2]);
  }
  mbar_wait(&bar[2], 0);
  tc::fence_after_sync();
  att_store_o(trow, l, valid, out + tok * D + head * ATT_HD);
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}

// ---- persistent, warp-specialised fused qkv + window attention ------------
// The same math as k_lt_attn_fused (identical MMA order per output element,
// so bit-identical results), restructured so the tensor core never waits on
// the SIMT phases of one work item (= GoP, 8x8 window, 64-dim head):
//   warp 0      TMA producer: per item 4 k-blocks of (2 token boxes of the
//               window + the head's 3 x 64 W_qkv rows) through a 2-stage ring;
//   warp 1      qkv GEMM issuer (runs up to two items ahead of the softmax);
//   warp 10     S = Q K^T / O = P V issuer (separate thread: neither issue
//               stream blocks the other);
//   warps 2-5,  two epilogue groups of 128 threads (one TMEM lane = one query
//   warps 6-9   row each); group b handles the items of parity b with its own
//               TMEM half (256 columns: qkv 0..191, S 0..127, O 128..191) and
//               its own operand tiles (Q, K, V; P over Q and K).
// TMEM per group: qkv columns 0..191, S 0..127 (over q|k, once they are in
// smem), O 192..255 -- so the projection of the group's next item only has
// to wait until this item's scores are consumed (p_ready), not for its O.
// Hand-offs are mbarriers: qkv_full / s_full / o_full (MMA commits),
// ops_ready / p_ready (128 epilogue arrivals each).
constexpr int AP_RING = 2 * AF_STAGE;                         // 80 KB
constexpr int AP_OPS = 3 * 16384;                             // Q, K, V per group
constexpr int AP_SMEM = AP_RING + 2 * AP_OPS + 256 + 1024;

__global__ void __launch_bounds__(352, 1)
    k_lt_attn_persist(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmW,
                      const float* __restrict__ bqkv, int G, int Ht, int Wt, int D,
                      __nv_bfloat16* __restrict__ out) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment by offset from smem_raw (keeps the shared address
  // space visible to the compiler: st.shared, not generic stores)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ops = smem + AP_RING;
  uint64_t* full = reinterpret_cast<uint64_t*>(ops + 2 * AP_OPS);
  uint64_t* empty = full + 2;
  uint64_t* qkv_full = empty + 2;     // [2] per group
  uint64_t* ops_ready = qkv_full + 2;
  uint64_t* s_full = ops_ready + 2;
  uint64_t* p_ready = s_full + 2;
  uint64_t* o_full = p_ready + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 2);

  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int wins_x = ceil_div(Wt, ATT_WIN);
  const int wins = ceil_div(Ht, ATT_WIN) * wins_x;
  const int heads = D / ATT_HD;
  const int n_items = G * wins * heads;
  // contiguous chunk of items per CTA (the 4 heads of a window back to back)
  const int per = ceil_div(n_items, (int)gridDim.x);
  const int it0 = blockIdx.x * per;
  const int n_my = max(0, min(n_items, it0 + per) - it0);
  const int ncb = D / BK;

  if (t == 0) {
    tc::prefetch_tmap(&tmH);
    tc::prefetch_tmap(&tmW);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&qkv_full[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&o_full[i], 1);
      mbar_init(&ops_ready[i], 128);
      mbar_init(&p_ready[i], 128);
    }
    fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  struct Item { int g, wy, wx, head; };
  auto item_coords = [=](int it) {
    Item c;
    c.head = it % heads;
    const int r = it / heads;
    const int win = r % wins;
    c.g = r / wins;
    c.wy = win / wins_x;
    c.wx = win - c.wy * wins_x;
    return c;
  };

  if (warp == 0) {
    // ---- TMA producer ----
    if (lane == 0) {
      int kb = 0;
      for (int i = 0; i < n_my; ++i) {
        const Item c = item_coords(it0 + i);
        const int g = c.g, wy = c.wy, wx = c.wx, head = c.head;
        for (int cb = 0; cb < ncb; ++cb, ++kb) {
          const int s = kb & 1;
          if (kb >= 2) mbar_wait(&empty[s], ((kb >> 1) - 1) & 1);
          uint8_t* st = smem + s * AF_STAGE;
          mbar_expect_tx(&full[s], AF_STAGE);
          tc::tma_load_5d(st, &tmH, cb * BK, wx * ATT_WIN, wy * ATT_WIN, 0, g, &full[s]);
          tc::tma_load_5d(st + 8192, &tmH, cb * BK, wx * ATT_WIN, wy * ATT_WIN, 1, g, &full[s]);
          for (int part = 0; part < 3; ++part)
            tc::tma_load_2d(st + 16384 + part * 8192, &tmW, cb * BK, part * D + head * ATT_HD,
                            &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ---- qkv projection issuer ----
    if (lane == 0) {
      constexpr uint32_t id0 = tc::idesc_bf16_f32(128, 192);
      int kb = 0;
      for (int i = 0; i < n_my; ++i) {
        const int b = i & 1;
        // TMEM columns 0..191 of group b are free once S(i-2) has been read
        // (p_ready(i-2)); O(i-2) lives in columns 192..255
        if (i >= 2) {
          mbar_wait(&p_ready[b], ((i >> 1) - 1) & 1);
          tc::fence_after_sync();
        }
        for (int cb = 0; cb < ncb; ++cb, ++kb) {
          const int s = kb & 1;
          mbar_wait(&full[s], (kb >> 1) & 1);
          tc::fence_after_sync();
          const uint64_t ad = tc::smem_desc_sw128(smem_u32(smem + s * AF_STAGE));
          const uint64_t bd = tc::smem_desc_sw128(smem_u32(smem + s * AF_STAGE + 16384));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            tc::mma_bf16(tmem + b * 256, ad + 2 * k, bd + 2 * k, id0, cb | k);
          tc::mma_commit(&empty[s]);
        }
        tc::mma_commit(&qkv_full[b]);
      }
    }
  } else if (warp == 10) {
    // ---- S = Q K^T and O = P V issuer ----
    if (lane == 0) {
      for (int i = 0; i < n_my; ++i) {
        const int b = i & 1, u = i >> 1;
        uint8_t* o = ops + b * AP_OPS;
        mbar_wait(&ops_ready[b], u & 1);
        tc::fence_after_sync();
        {
          constexpr uint32_t id1 = tc::idesc_bf16_f32(128, 128);
          const uint64_t ad = tc::smem_desc_sw128(smem_u32(o));
          const uint64_t bd = tc::smem_desc_sw128(smem_u32(o + 16384));
#pragma unroll
          for (int k = 0; k < 4; ++k) tc::mma_bf16(tmem + b * 256, ad + 2 * k, bd + 2 * k, id1, k);
          tc::mma_commit(&s_full[b]);
        }
        mbar_wait(&p_ready[b], u & 1);
        tc::fence_after_sync();
        att_issue_pv(tmem + b * 256 + 192, o, o + 32768);
        tc::mma_commit(&o_full[b]);
      }
    }
  } else {
    // ---- epilogue groups ----
    const int grp = (warp - 2) >> 2;
    const int q = ((warp & 3) << 5) | lane;          // TMEM lane = query / token row
    const int ft = q >> 6, lt = q & 63;
    uint8_t* o = ops + grp * AP_OPS;
    uint8_t* sQ = o;
    uint8_t* sK = o + 16384;
    uint8_t* sV = o + 32768;
    const uint32_t tb = tmem + grp * 256 + ((uint32_t)((warp & 3) * 32) << 16);
    for (int i = grp; i < n_my; i += 2) {
      const int u = i >> 1;
      const Item c = item_coords(it0 + i);
      const int g = c.g, wy = c.wy, wx = c.wx, head = c.head;
      const int y = wy * ATT_WIN + (lt >> 3), x = wx * ATT_WIN + (lt & 7);
      const bool valid = y < Ht && x < Wt;
      // -- qkv: +bias, bf16; Q, K and V rows into their tiles --
      mbar_wait(&qkv_full[grp], u & 1);
      tc::fence_after_sync();
      att_qkv_epilogue(tb, bqkv, D, head, valid, q, sQ, sK, sV);
      fence_proxy_async_smem();
      tc::fence_before_sync();
      tc::mbar_arrive(&ops_ready[grp]);
      // -- softmax of this query row --
      mbar_wait(&s_full[grp], u & 1);
      tc::fence_after_sync();
      const uint32_t vrow = (1u << min(8, Ht - wy * ATT_WIN)) - 1u;
      const uint32_t vcol = (1u << min(8, Wt - wx * ATT_WIN)) - 1u;
      // P over Q and K (the S GEMM that read them has completed: s_full)
      const float l = att_softmax_p(tb, o, q, vrow, vcol);
      fence_proxy_async_smem();
      tc::fence_before_sync();
      tc::mbar_arrive(&p_ready[grp]);
      // -- O / l --
      mbar_wait(&o_full[grp], u & 1);
      tc::fence_after_sync();
      const size_t tok = (((size_t)g * 2 + ft) * Ht + y) * Wt + x;
      att_store_o(tb + 192, l, valid, out + tok * D + head * ATT_HD);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

// ---- downscale + pad + patchify --------------------------------------------
template <int S>
__global__ void k_lt_patchify(const float* __restrict__ src, int G, int H, int W, int h, int w,
                              int Ht, int Wt, __nv_bfloat16* __restrict__ pI,
                              __nv_bfloat16* __restrict__ pP) {
  // grid: x = 256-pixel column tiles of a padded row, y = padded row,
  // z = frame (g * 9 + f): no 64-bit index divisions per pixel
  const int PW = Wt * 8;
  const int X = blockIdx.x * blockDim.x + threadIdx.x;
  if (X >= PW) return;
  const int Y = blockIdx.y;
  const int f = (int)(blockIdx.z % 9);
  const int g = (int)(blockIdx.z / 9);
  const int xc = min(X, w - 1), yc = min(Y, h - 1);  // np.pad(mode="edge") of the working frame
  const float* fr = src + ((int64_t)g * 9 + f) * (int64_t)H * W * 3;
  float px[3];
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const int rr = min(yc * S + j, H - 1);
#pragma unroll
      for (int l = 0; l < S; ++l) {
        const int cc = min(xc * S + l, W - 1);
        acc = acc + (double)__ldg(fr + ((int64_t)rr * W + cc) * 3 + ch);
      }
    }
    px[ch] = __double2float_rn(acc / (double)(S * S));
  }
  const int ty = Y >> 3, py = Y & 7, tx = X >> 3, pxl = X & 7;
  __nv_bfloat16* dst;
  if (f == 0)
    dst = pI + ((int64_t)(g * Ht + ty) * Wt + tx) * 192 + (py * 8 + pxl) * 3;
  else
    dst = pP + ((int64_t)(g * Ht + ty) * Wt + tx) * 1536 + (((f - 1) * 8 + py) * 8 + pxl) * 3;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) dst[ch] = __float2bfloat16_rn(px[ch]);
}

// ---- mask-aware decoder input ----------------------------------------------
__global__ void k_lt_dec_in(const double* __restrict__ tok, const uint8_t* __restrict__ mask, int G,
                            int Ht, int Wt, __nv_bfloat16* __restrict__ out) {
  const int64_t n = (int64_t)Ht * Wt;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)G * 2 * n) return;
  const int64_t pos = idx % n;
  const int64_t gt = idx / n;
  const int t = (int)(gt % 2);
  const int64_t g = gt / 2;
  int64_t src = idx;
  if (t == 1 && !mask[idx]) src = (g * 2) * n + pos;  // conceal P with the co-located I token
  const bool ok = mask[src] != 0;
  uint4 o[DEC_IN_C / 8];
#pragma unroll
  for (int q = 0; q < DEC_IN_C / 8; ++q) o[q] = make_uint4(0, 0, 0, 0);
  if (ok) {
    __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(o);
#pragma unroll
    for (int i = 0; i < FSQ_C; ++i) {
      const int L = fsq_levels(i), hw = L / 2;
      double q = rint(tok[src * FSQ_C + i] * (double)hw);
      q = fmin(fmax(q, (double)-hw), (double)(L - 1 - hw));
      ob[i] = __float2bfloat16_rn((float)(q / (double)hw));
    }
  }
  uint4* op = reinterpret_cast<uint4*>(out + idx * DEC_IN_C);
#pragma unroll
  for (int q = 0; q < DEC_IN_C / 8; ++q) op[q] = o[q];
}

template <int BN, int EPI, int NST>
static int launch_conv_n(const SstConvDesc* d, cudaStream_t st) {
  using Cfg = TileCfg<BN, NST>;
  if (d->N % BN != 0) return SST_ERR_ARG;
  CUtensorMap tmA, tmB, tmC;
  memset(&tmA, 0, sizeof(tmA));
  memset(&tmB, 0, sizeof(tmB));
  memset(&tmC, 0, sizeof(tmC));
  const uint64_t adims[5] = {(uint64_t)d->in_C, (uint64_t)d->in_W, (uint64_t)d->in_H,
                             (uint64_t)d->in_T, (uint64_t)d->G};
  if (!make_tmap_bf16_5d(&tmA, d->in, adims, BOX_X, BOX_Y)) return SST_ERR_ARG;
  if (!make_tmap_bf16_2d(&tmB, d->weight, (uint64_t)d->K, (uint64_t)d->N, BN)) return SST_ERR_ARG;
  if (EPI == SST_LT_EPI_STORE) {
    const uint64_t cdims[5] = {(uint64_t)d->N, (uint64_t)d->Wt, (uint64_t)d->Ht,
                               (uint64_t)d->out_T, (uint64_t)d->G};
    if (!make_tmap_bf16_5d(&tmC, d->out, cdims, BOX_X, BOX_Y)) return SST_ERR_ARG;
  }
  ConvArgs a;
  memset(&a, 0, sizeof(a));
  a.Ht = d->Ht; a.Wt = d->Wt;
  a.tiles_x = ceil_div(d->Wt, BOX_X);
  a.tiles_y = ceil_div(d->Ht, BOX_Y);
  a.t_lo = d->t_lo; a.t_cnt = d->t_cnt;
  a.n_taps = d->n_taps;
  a.kb_per_tap = d->in_C / BK;
  a.N = d->N;
  a.out_T = d->out_T;
  for (int i = 0; i < d->n_taps; ++i)
    for (int j = 0; j < 3; ++j) a.taps[i][j] = (signed char)d->taps[i][j];
  a.bias = d->bias;
  a.act = d->act;
  a.residual = static_cast<const __nv_bfloat16*>(d->residual);
  a.codes = d->codes; a.idx = d->idx; a.mask = d->mask;
  a.frames = d->frames; a.h = d->h; a.w = d->w; a.frame_base = d->frame_base;
  const int64_t mt = (int64_t)d->G * d->t_cnt * a.tiles_y * a.tiles_x;
  if (mt <= 0 || mt > 0x7fffffff) return SST_ERR_ARG;
  dim3 grid((unsigned)mt, d->N / BN);
  auto kern = k_lt_conv<BN, EPI, NST>;
  SST_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  kern<<<grid, 128, Cfg::SMEM, st>>>(tmA, tmB, tmC, a);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

template <int BN, int EPI>
static int launch_conv(const SstConvDesc* d, cudaStream_t st) {
  if (d->n_taps * (d->in_C / BK) <= 8) return launch_conv_n<BN, EPI, 2>(d, st);
  return launch_conv_n<BN, EPI, 4>(d, st);
}

static bool is_taps233(const SstConvDesc* d) {
  if (d->n_taps != 18) return false;
  for (int i = 0; i < 18; ++i) {
    const int kt = i / 9, ky = (i / 3) % 3, kx = i % 3;
    if (d->taps[i][0] != kt - 1 || d->taps[i][1] != ky - 1 || d->taps[i][2] != kx - 1) return false;
  }
  return true;
}

static int launch_conv233p(const SstConvDesc* d, cudaStream_t st) {
  if (d->N % c233p::BN != 0 || d->t_lo != 0 || d->t_cnt != d->in_T || d->in_T != d->out_T ||
      d->in_W != d->Wt || d->in_H != d->Ht)
    return SST_ERR_ARG;
  CUtensorMap tmA, tmB;
  memset(&tmA, 0, sizeof(tmA));
  memset(&tmB, 0, sizeof(tmB));
  const uint64_t adims[5] = {(uint64_t)d->in_C, (uint64_t)d->in_W, (uint64_t)d->in_H,
                             (uint64_t)d->in_T, (uint64_t)d->G};
  if (!make_tmap_bf16_5d(&tmA, d->in, adims, c233p::PITCH, c233p::HROWS)) return SST_ERR_ARG;
  if (!make_tmap_bf16_2d(&tmB, d->weight, (uint64_t)d->K, (uint64_t)d->N, c233p::BN))
    return SST_ERR_ARG;
  ConvArgs a;
  memset(&a, 0, sizeof(a));
  a.Ht = d->Ht; a.Wt = d->Wt;
  a.tiles_x = ceil_div(d->Wt, c233p::TILE);
  a.tiles_y = ceil_div(d->Ht, c233p::TILE);
  a.t_lo = 0; a.t_cnt = d->t_cnt;
  a.n_taps = 18;
  a.kb_per_tap = d->in_C / BK;
  a.N = d->N;
  a.out_T = d->out_T;
  a.bias = d->bias;
  a.act = d->act;
  a.residual = static_cast<const __nv_bfloat16*>(d->residual);
  a.out = static_cast<__nv_bfloat16*>(d->out);
  const int n_halves = d->N / c233p::BN;
  const int64_t units = (int64_t)d->G * d->t_cnt * a.tiles_y * a.tiles_x * n_halves;
  if (units <= 0 || units > 0x7fffffff) return SST_ERR_ARG;
  int n_sm = 0, dev = 0;                     // the current device's SM count (per call:
  SST_CUDA_TRY(cudaGetDevice(&dev));         // a process may drive several devices)
  SST_CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  const int grid = (int)(units < n_sm ? units : n_sm);
  SST_CUDA_TRY(cudaFuncSetAttribute(k_lt_conv233p, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    c233p::SMEM));
  k_lt_conv233p<<<grid, c233p::THREADS, c233p::SMEM, st>>>(tmA, tmB, a, (int)units, n_halves);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

static int launch_convpair_pixels(const SstConvDesc* d, cudaStream_t st) {
  if (d->N % 192 != 0 || d->n_taps != 1 || d->taps[0][1] != 0 || d->taps[0][2] != 0 ||
      d->in_W != d->Wt || d->in_H != d->Ht)
    return SST_ERR_ARG;
  CUtensorMap tmA, tmB, tmC;
  memset(&tmA, 0, sizeof(tmA));
  memset(&tmB, 0, sizeof(tmB));
  memset(&tmC, 0, sizeof(tmC));
  const uint64_t adims[5] = {(uint64_t)d->in_C, (uint64_t)d->in_W, (uint64_t)d->in_H,
                             (uint64_t)d->in_T, (uint64_t)d->G};
  if (!make_tmap_bf16_5d(&tmA, d->in, adims, 8, 16)) return SST_ERR_ARG;
  if (!make_tmap_bf16_2d(&tmB, d->weight, (uint64_t)d->K, (uint64_t)d->N, 96)) return SST_ERR_ARG;
  ConvArgs a;
  memset(&a, 0, sizeof(a));
  a.Ht = d->Ht; a.Wt = d->Wt;
  a.tiles_x = ceil_div(d->Wt, c233c::TILE);
  a.tiles_y = ceil_div(d->Ht, c233c::TILE);
  a.t_lo = d->t_lo; a.t_cnt = d->t_cnt;
  a.n_taps = 1;
  for (int j = 0; j < 3; ++j) a.taps[0][j] = (signed char)d->taps[0][j];
  a.kb_per_tap = d->in_C / BK;
  a.N = d->N;
  a.out_T = d->out_T;
  a.bias = d->bias;
  a.frames = d->frames; a.h = d->h; a.w = d->w; a.frame_base = d->frame_base;
  const int n_blocks = d->N / 192;
  const int64_t units = (int64_t)d->G * d->t_cnt * a.tiles_y * a.tiles_x * n_blocks;
  if (units <= 0 || units > 0x7fffffff) return SST_ERR_ARG;
  int n_sm = 0, dev = 0;
  SST_CUDA_TRY(cudaGetDevice(&dev));
  SST_CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  const int64_t pairs = units < n_sm / 2 ? units : n_sm / 2;
  auto kern = k_lt_convpair<false, false, true>;
  const int smem = pair_smem<false, false, true>();
  SST_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<(unsigned)(2 * pairs), c233c::THREADS, smem, st>>>(tmA, tmB, tmC, a, (int)units, n_blocks);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

static int launch_convpair(const SstConvDesc* d, cudaStream_t st, bool halo) {
  if (d->N % 256 != 0 || d->in_W != d->Wt || d->in_H != d->Ht) return SST_ERR_ARG;
  if (halo && (d->t_lo != 0 || d->t_cnt != d->in_T || d->in_T != d->out_T)) return SST_ERR_ARG;
  if (!halo && (d->n_taps != 1 || d->taps[0][1] != 0 || d->taps[0][2] != 0)) return SST_ERR_ARG;
  CUtensorMap tmA, tmB;
  memset(&tmA, 0, sizeof(tmA));
  memset(&tmB, 0, sizeof(tmB));
  const uint64_t adims[5] = {(uint64_t)d->in_C, (uint64_t)d->in_W, (uint64_t)d->in_H,
                             (uint64_t)d->in_T, (uint64_t)d->G};
  if (!make_tmap_bf16_5d(&tmA, d->in, adims, halo ? c233c::PITCH : 8, halo ? c233c::HROWS : 16))
    return SST_ERR_ARG;
  if (!make_tmap_bf16_2d(&tmB, d->weight, (uint64_t)d->K, (uint64_t)d->N, c233c::BNH))
    return SST_ERR_ARG;
  ConvArgs a;
  memset(&a, 0, sizeof(a));
  a.Ht = d->Ht; a.Wt = d->Wt;
  a.tiles_x = ceil_div(d->Wt, c233c::TILE);
  a.tiles_y = ceil_div(d->Ht, c233c::TILE);
  a.t_lo = d->t_lo; a.t_cnt = d->t_cnt;
  a.n_taps = d->n_taps;
  for (int i = 0; i < d->n_taps; ++i)
    for (int j = 0; j < 3; ++j) a.taps[i][j] = (signed char)d->taps[i][j];
  a.kb_per_tap = d->in_C / BK;
  a.N = d->N;
  a.out_T = d->out_T;
  a.bias = d->bias;
  a.act = d->act;
  a.residual = static_cast<const __nv_bfloat16*>(d->residual);
  a.out = static_cast<__nv_bfloat16*>(d->out);
  const int n_blocks = d->N / 256;
  const int64_t units = (int64_t)d->G * d->t_cnt * a.tiles_y * a.tiles_x * n_blocks;
  if (units <= 0 || units > 0x7fffffff) return SST_ERR_ARG;
  int n_sm = 0, dev = 0;                     // the current device's SM count (per call:
  SST_CUDA_TRY(cudaGetDevice(&dev));         // a process may drive several devices)
  SST_CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  const int64_t pairs = units < n_sm / 2 ? units : n_sm / 2;
  CUtensorMap tmC;
  memset(&tmC, 0, sizeof(tmC));
  const bool tma_store = !halo;
  if (tma_store) {
    const uint64_t cdims[5] = {(uint64_t)d->N, (uint64_t)d->Wt, (uint64_t)d->Ht,
                               (uint64_t)d->out_T, (uint64_t)d->G};
    if (!make_tmap_bf16_5d(&tmC, d->out, cdims, 8, 16)) return SST_ERR_ARG;
  }
  auto kern = halo ? k_lt_convpair<true, false> : k_lt_convpair<false, true>;
  const int smem = halo ? pair_smem<true, false>() : pair_smem<false, true>();
  SST_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<(unsigned)(2 * pairs), c233c::THREADS, smem, st>>>(tmA, tmB, tmC, a, (int)units, n_blocks);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

static int launch_conv233(const SstConvDesc* d, cudaStream_t st) {
  if (d->N % c233::BN != 0 || d->t_lo != 0 || d->t_cnt != d->in_T || d->in_T != d->out_T ||
      d->in_W != d->Wt || d->in_H != d->Ht)
    return SST_ERR_ARG;
  CUtensorMap tmA, tmB;
  memset(&tmA, 0, sizeof(tmA));
  memset(&tmB, 0, sizeof(tmB));
  const uint64_t adims[5] = {(uint64_t)d->in_C, (uint64_t)d->in_W, (uint64_t)d->in_H,
                             (uint64_t)d->in_T, (uint64_t)d->G};
  if (!make_tmap_bf16_5d(&tmA, d->in, adims, c233::PITCH, c233::HROWS)) return SST_ERR_ARG;
  if (!make_tmap_bf16_2d(&tmB, d->weight, (uint64_t)d->K, (uint64_t)d->N, c233::BN)) return SST_ERR_ARG;
  ConvArgs a;
  memset(&a, 0, sizeof(a));
  a.Ht = d->Ht; a.Wt = d->Wt;
  a.tiles_x = ceil_div(d->Wt, c233::TILE);
  a.tiles_y = ceil_div(d->Ht, c233::TILE);
  a.t_lo = 0; a.t_cnt = d->t_cnt;
  a.n_taps = 18;
  a.kb_per_tap = d->in_C / BK;
  a.N = d->N;
  a.out_T = d->out_T;
  a.bias = d->bias;
  a.act = d->act;
  a.residual = static_cast<const __nv_bfloat16*>(d->residual);
  a.out = static_cast<__nv_bfloat16*>(d->out);
  const int64_t mt = (int64_t)d->G * d->t_cnt * a.tiles_y * a.tiles_x;
  if (mt <= 0 || mt > 0x7fffffff) return SST_ERR_ARG;
  dim3 grid((unsigned)mt, d->N / c233::BN);
  SST_CUDA_TRY(cudaFuncSetAttribute(k_lt_conv233, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    c233::SMEM));
  k_lt_conv233<<<grid, c233::THREADS, c233::SMEM, st>>>(tmA, tmB, a);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

}  // namespace lt
}  // namespace sst

#include <cstdlib>

using namespace sst;

extern "C" int sst_lt_conv(const SstConvDesc* d, void* stream) {
  if (!d || !d->in || !d->weight || !d->bias) return SST_ERR_ARG;
  if (reinterpret_cast<uintptr_t>(d->bias) & 15u) return SST_ERR_ARG;   // float4 bias loads
  if (d->in_C <= 0 || d->in_C % lt::BK != 0) return SST_ERR_ARG;
  if (d->n_taps < 1 || d->n_taps > 27 || d->K != d->n_taps * d->in_C) return SST_ERR_ARG;
  if (d->G <= 0 || d->Ht <= 0 || d->Wt <= 0 || d->t_cnt <= 0) return SST_ERR_ARG;
  for (int i = 0; i < d->n_taps; ++i)
    for (int j = 0; j < 3; ++j)
      if (d->taps[i][j] < -8 || d->taps[i][j] > 8) return SST_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (d->epi) {
    case SST_LT_EPI_STORE: {
      if (!d->out || d->act < 0 || d->act > 1) return SST_ERR_ARG;
      // Default for the causal (2,3,3) convs: the CTA-pair kernel (N = 256) or
      // the persistent single-CTA kernel (other N).  A/B switches:
      // SST_LT_CONV=persistent / halo (non-persistent) / generic (per-tap loads)
      const char* mode = getenv("SST_LT_CONV");
      const bool generic = mode && mode[0] == 'g';
      const bool halo1 = mode && mode[0] == 'h';
      const bool single = mode && mode[0] == 'p';
      if (!generic && lt::is_taps233(d) && d->N % lt::c233::BN == 0) {
        if (!single && !halo1 && d->N % 256 == 0) return lt::launch_convpair(d, st, true);
        return halo1 ? lt::launch_conv233(d, st) : lt::launch_conv233p(d, st);
      }
      // long-K 1x1 layers (K >= 1024: the P patch embedding) with N % 256 == 0:
      // the CTA-pair kernel without halo.  Short-K 1x1 layers (qkv / proj,
      // K = 256) are store-bound and keep the tile kernel's swizzled TMA-store
      // epilogue (measured: qkv 0.30 ms tile kernel vs 0.46 ms pair kernel).
      if (!generic && d->n_taps == 1 && d->taps[0][1] == 0 && d->taps[0][2] == 0 &&
          d->N % 256 == 0 && d->in_W == d->Wt && d->in_H == d->Ht) {
        const char* m1 = getenv("SST_LT_GEMM");
        if (!(m1 && m1[0] == 't')) return lt::launch_convpair(d, st, false);
      }
      return lt::launch_conv<128, SST_LT_EPI_STORE>(d, st);
    }
    case SST_LT_EPI_FSQ:
      if (!d->codes || !d->idx || !d->mask || d->N != 16 || d->t_lo != 0 || d->t_cnt != 2)
        return SST_ERR_ARG;
      return lt::launch_conv<16, SST_LT_EPI_FSQ>(d, st);
    case SST_LT_EPI_PIXELS: {
      if (!d->frames || d->h <= 0 || d->w <= 0 || d->frame_base < 0 ||
          d->frame_base + d->N / 192 > 9 || d->h > d->Ht * 8 || d->w > d->Wt * 8)
        return SST_ERR_ARG;
      const char* m2 = getenv("SST_LT_GEMM");          // "tile": the per-tile kernel (A/B)
      if (!(m2 && m2[0] == 't') && d->N % 192 == 0 && d->n_taps == 1 && d->taps[0][1] == 0 &&
          d->taps[0][2] == 0 && d->in_W == d->Wt && d->in_H == d->Ht)
        return lt::launch_convpair_pixels(d, st);
      return lt::launch_conv<192, SST_LT_EPI_PIXELS>(d, st);
    }
    default:
      return SST_ERR_ARG;
  }
}

extern "C" int sst_lt_patchify(const float* frames, int G, int H, int W, int s, void* pI, void* pP,
                               void* stream) {
  if (!frames || !pI || !pP || G <= 0 || H <= 0 || W <= 0) return SST_ERR_ARG;
  if (s < 1 || s > 3) return SST_ERR_ARG;
  const int h = ceil_div(H, s), w = ceil_div(W, s);
  const int Ht = ceil_div(h, 8), Wt = ceil_div(w, 8);
  const int threads = 256;
  if ((int64_t)G * 9 > 65535 || Ht * 8 > 65535) return SST_ERR_ARG;
  const dim3 blocks(ceil_div(Wt * 8, threads), Ht * 8, G * 9);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto* i = static_cast<__nv_bfloat16*>(pI);
  auto* p = static_cast<__nv_bfloat16*>(pP);
  switch (s) {
    case 1: lt::k_lt_patchify<1><<<blocks, threads, 0, st>>>(frames, G, H, W, h, w, Ht, Wt, i, p); break;
    case 2: lt::k_lt_patchify<2><<<blocks, threads, 0, st>>>(frames, G, H, W, h, w, Ht, Wt, i, p); break;
    default: lt::k_lt_patchify<3><<<blocks, threads, 0, st>>>(frames, G, H, W, h, w, Ht, Wt, i, p); break;
  }
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_lt_dec_in(const double* tok, const uint8_t* mask, int G, int Ht, int Wt, void* out,
                             void* stream) {
  if (!tok || !mask || !out || G <= 0 || Ht <= 0 || Wt <= 0) return SST_ERR_ARG;
  const int64_t total = (int64_t)G * 2 * Ht * Wt;
  const int threads = 256;
  lt::k_lt_dec_in<<<(unsigned)ceil_div64(total, threads), threads, 0,
                    static_cast<cudaStream_t>(stream)>>>(tok, mask, G, Ht, Wt,
                                                         static_cast<__nv_bfloat16*>(out));
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_lt_attn(const void* qkv, int G, int Ht, int Wt, int D, void* out, void* stream) {
  if (!qkv || !out || G <= 0 || Ht <= 0 || Wt <= 0 || D <= 0 || D % lt::ATT_HD) return SST_ERR_ARG;
  if (G > 65535 || D / lt::ATT_HD > 65535) return SST_ERR_ARG;
  const int64_t wins = (int64_t)ceil_div(Ht, lt::ATT_WIN) * ceil_div(Wt, lt::ATT_WIN);
  if (wins > 0x7fffffff) return SST_ERR_ARG;
  dim3 grid((unsigned)wins, D / lt::ATT_HD, G);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const char* mode = getenv("SST_LT_ATTN");          // "simt": the SIMT core (A/B)
  if (mode && mode[0] == 's') {
    const int smem = 2 * 128 * lt::ATT_HD * 4 + 128 * 4;
    SST_CUDA_TRY(cudaFuncSetAttribute(lt::k_lt_attn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    lt::k_lt_attn<<<grid, 128, smem, st>>>(static_cast<const __nv_bfloat16*>(qkv), G, Ht, Wt, D,
                                           static_cast<__nv_bfloat16*>(out));
  } else {
    SST_CUDA_TRY(cudaFuncSetAttribute(lt::k_lt_attn_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      lt::ATT_SMEM));
    lt::k_lt_attn_tc<<<grid, 128, lt::ATT_SMEM, st>>>(static_cast<const __nv_bfloat16*>(qkv), G, Ht,
                                                       Wt, D, static_cast<__nv_bfloat16*>(out));
  }
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_lt_attn_fused(const void* h, const void* w_qkv, const float* b_qkv, int G, int Ht,
                                 int Wt, int D, void* out, void* stream) {
  if (!h || !w_qkv || !b_qkv || !out || G <= 0 || Ht <= 0 || Wt <= 0 || D <= 0) return SST_ERR_ARG;
  if (reinterpret_cast<uintptr_t>(b_qkv) & 15u) return SST_ERR_ARG;   // float4 bias loads
  if (D % lt::ATT_HD || G > 65535 || D / lt::ATT_HD > 65535) return SST_ERR_ARG;
  const int64_t wins = (int64_t)ceil_div(Ht, lt::ATT_WIN) * ceil_div(Wt, lt::ATT_WIN);
  if (wins > 0x7fffffff) return SST_ERR_ARG;
  CUtensorMap tmH, tmW;
  memset(&tmH, 0, sizeof(tmH));
  memset(&tmW, 0, sizeof(tmW));
  const uint64_t hdims[5] = {(uint64_t)D, (uint64_t)Wt, (uint64_t)Ht, 2, (uint64_t)G};
  if (!make_tmap_bf16_5d(&tmH, h, hdims, lt::ATT_WIN, lt::ATT_WIN)) return SST_ERR_ARG;
  if (!make_tmap_bf16_2d(&tmW, w_qkv, (uint64_t)D, (uint64_t)(3 * D), lt::ATT_HD)) return SST_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // default: the persistent warp-specialised kernel (0.211 ms at the learned
  // leg's shape, 32 x 1080p GoPs, D=256; scripts/attn_micro.py).
  // SST_LT_ATTN=fused: one CTA per (GoP, window, head), two CTAs per SM
  // (0.257 ms) -- bit-identical.  Both are bound by the SIMT epilogue; the
  // persistent kernel overlaps it with the next item's qkv GEMM.
  const char* ea = getenv("SST_LT_ATTN");
  if (!(ea && !strcmp(ea, "fused"))) {
    const int64_t items = wins * (D / lt::ATT_HD) * (int64_t)G;
    if (items > 0x7fffffff) return SST_ERR_ARG;
    int dev = 0, sms = 148;
    SST_CUDA_TRY(cudaGetDevice(&dev));
    SST_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int grid = (int)(items < sms ? items : sms);
    SST_CUDA_TRY(cudaFuncSetAttribute(lt::k_lt_attn_persist,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, lt::AP_SMEM));
    lt::k_lt_attn_persist<<<grid, 352, lt::AP_SMEM, st>>>(tmH, tmW, b_qkv, G, Ht, Wt, D,
                                                          static_cast<__nv_bfloat16*>(out));
    SST_LAUNCH_CHECK();
    return SST_OK;
  }
  dim3 grid((unsigned)wins, D / lt::ATT_HD, G);
  SST_CUDA_TRY(cudaFuncSetAttribute(lt::k_lt_attn_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    lt::AF_SMEM));
  lt::k_lt_attn_fused<<<grid, 128, lt::AF_SMEM, st>>>(tmH, tmW, b_qkv, G, Ht, Wt, D,
                                                      static_cast<__nv_bfloat16*>(out));
  SST_LAUNCH_CHECK();
  return SST_OK;
}
