// Int8 learned tokenizer (learned_i8.py): the plug-in
// network on tcgen05.mma .kind::i8 -- int8 activations and weights, int32
// accumulators in TMEM.  Every result is exact integer arithmetic, so the
// kernels agree bit for bit with oracle/learned_i8_oracle.py (which defines
// the arithmetic) regardless of summation order.
//
//   k_l8_patchify  box downscale (bit-exact, codec.py:202-214) + edge pad +
//                  8x8(x8) patchify -> int8 rint(px * 255) - 128
//   k_l8_patchify_haar  the same through the integer 3-D Haar front end
//   k_l8_tile      generic implicit-GEMM layer: one CTA = 128 tokens (16x8)
//                  x BN channels, per-tap 5-D TMA loads, 4-stage ring; STORE
//                  (requantise + SiLU table + saturating residual), FSQ head
//                  and PIXELS epilogues
//   k_l8_pair      the CTA-pair (cta_group::2) layer for N % 256 == 0 (and
//                  the 192-column pixel units): causal (2,3,3) convs with
//                  one TMA halo per (temporal tap, 128-channel block) shared
//                  by the 9 spatial taps, or 1x1 GEMMs with a TMA-store
//                  epilogue; M = 256 x N = 256 x K = 32 per instruction
//   k_l8_attn      causal 8x8-window attention, 128-dim heads: S = Q K^T and
//                  O = P V on tcgen05 (kind::i8, P unsigned), integer softmax
//                  (uint8 exp table, exact row sums, floor-rounded division)
//
// Byte layout of an int8 K-major operand tile = that of the bf16 kernels
// (learned.cu): 128-byte swizzled rows; one MMA eats K = 32 int8 = 32 bytes,
// so a 128-byte K block is 4 instructions, as for bf16 -- at twice the K.
#include <cuda_runtime.h>
#include <cstring>

#include "common.cuh"
#include "tc.cuh"

namespace sst {
namespace l8 {

constexpr int KB = 128;            // int8 channels per 128-byte K block
constexpr int BM = 128;            // tokens per tile kernel CTA (16 x 8 box)
constexpr int BOX_X = 16, BOX_Y = 8;
constexpr int A_BYTES = BM * KB;   // 16 KB
constexpr int FSQ_C = 12;

__device__ __forceinline__ int fsq_levels(int i) { return (i % 6) < 3 ? 8 : 5; }
__device__ __forceinline__ int fsq_basis(int i) {
  const int j = i % 6;
  return j == 0 ? 1 : j == 1 ? 8 : j == 2 ? 64 : j == 3 ? 512 : j == 4 ? 2560 : 12800;
}

struct Args {
  int Ht, Wt, tiles_x, tiles_y, t_lo, t_cnt;
  int n_taps, kb_per_tap, N, out_T;
  signed char taps[27][3];
  const int32_t* bias;
  int shift, act;
  const int8_t* lut;
  const int8_t* residual;
  int8_t* out;
  double* codes;
  int32_t* idx;
  uint8_t* mask;
  float* frames;               // PIXELS: float32 frames, or uint8 q frames when pix_u8
  int h, w, frame_base;
  int pix_u8;
};

__device__ __forceinline__ int rq(int32_t acc, int32_t b, int sh) {
  const int v = (acc + b + (1 << (sh - 1))) >> sh;      // arithmetic shift: floor
  return min(max(v, -127), 127);
}

__device__ __forceinline__ uint32_t pack4(int a, int b, int c, int d) {
  return (uint32_t)(a & 0xFF) | ((uint32_t)(b & 0xFF) << 8) | ((uint32_t)(c & 0xFF) << 16) |
         ((uint32_t)(d & 0xFF) << 24);
}

// bytes (a, b, c, d) = sat_s8(a .. d), a lowest: two cvt.pack.sat (I2IP), the
// saturation doing the upper clamp of a requantisation for free
__device__ __forceinline__ uint32_t pack4_sat(int a, int b, int c, int d) {
  uint32_t hi, r;
  asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(hi) : "r"(d), "r"(c));
  asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(b), "r"(a), "r"(hi));
  return r;
}

// bytes = sat_u8 of four int32 (clamp to [0, 255] in the pack)
__device__ __forceinline__ uint32_t pack4_satu8(int a, int b, int c, int d) {
  uint32_t hi, r;
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, 0;" : "=r"(hi) : "r"(d), "r"(c));
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(b), "r"(a), "r"(hi));
  return r;
}

// requantise without the upper clamp (pack4_sat saturates at 127)
__device__ __forceinline__ int rq_lo(int32_t acc, int32_t b_rnd, int sh) {
  return max((acc + b_rnd) >> sh, -127);
}

// STORE epilogue of 32 accumulator columns (n0 .. n0+31): requantise, SiLU
// table, saturating residual add; 32 int8 results packed into o[0..1].
__device__ __forceinline__ void epi_store32(const float (&acc)[32], const Args& a, int n0,
                                            const uint4* res, uint4 (&o)[2]) {
  int y[32];
  const int4* bp = reinterpret_cast<const int4*>(a.bias + n0);
  if (!a.act && res == nullptr) {
    // plain requantisation: add, shift, lower clamp; the upper clamp is the
    // pack's saturation
    const int rnd = 1 << (a.shift - 1);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      uint32_t wd[4];
#pragma unroll
      for (int i4 = 0; i4 < 4; ++i4) {
        const int4 bb = __ldg(bp + q * 4 + i4);
        const int j = q * 16 + 4 * i4;
        wd[i4] = pack4_sat(rq_lo(__float_as_int(acc[j + 0]), bb.x + rnd, a.shift),
                           rq_lo(__float_as_int(acc[j + 1]), bb.y + rnd, a.shift),
                           rq_lo(__float_as_int(acc[j + 2]), bb.z + rnd, a.shift),
                           rq_lo(__float_as_int(acc[j + 3]), bb.w + rnd, a.shift));
      }
      o[q] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    }
    return;
  }
#pragma unroll
  for (int i4 = 0; i4 < 8; ++i4) {
    const int4 bb = __ldg(bp + i4);
    y[4 * i4 + 0] = rq(__float_as_int(acc[4 * i4 + 0]), bb.x, a.shift);
    y[4 * i4 + 1] = rq(__float_as_int(acc[4 * i4 + 1]), bb.y, a.shift);
    y[4 * i4 + 2] = rq(__float_as_int(acc[4 * i4 + 2]), bb.z, a.shift);
    y[4 * i4 + 3] = rq(__float_as_int(acc[4 * i4 + 3]), bb.w, a.shift);
  }
  if (a.act) {
#pragma unroll
    for (int i = 0; i < 32; ++i) y[i] = __ldg(a.lut + y[i] + 128);
  }
  if (res != nullptr) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint4 u = res[q];
      const uint32_t wds[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int wi = 0; wi < 4; ++wi)
#pragma unroll
        for (int bi = 0; bi < 4; ++bi) {
          const int r = (int)(int8_t)((wds[wi] >> (8 * bi)) & 0xFF);
          int& v = y[q * 16 + wi * 4 + bi];
          v = min(max(r + v, -127), 127);
        }
    }
  }
#pragma unroll
  for (int q = 0; q < 2; ++q)   // values in [-127, 127]: the saturating pack is exact
    o[q] = make_uint4(pack4_sat(y[q * 16 + 0], y[q * 16 + 1], y[q * 16 + 2], y[q * 16 + 3]),
                      pack4_sat(y[q * 16 + 4], y[q * 16 + 5], y[q * 16 + 6], y[q * 16 + 7]),
                      pack4_sat(y[q * 16 + 8], y[q * 16 + 9], y[q * 16 + 10], y[q * 16 + 11]),
                      pack4_sat(y[q * 16 + 12], y[q * 16 + 13], y[q * 16 + 14], y[q * 16 + 15]));
}

__device__ __forceinline__ float pixel(int32_t acc, int32_t b, int sh) {
  int v = (acc + b + (1 << (sh - 1))) >> sh;
  v = min(max(v, 0), 255);
  return __fdiv_rn((float)v, 255.0f);
}

// the same through a 256-entry table of q / 255 (filled with __fdiv_rn, so
// identical values; one shared load instead of an IEEE division per sample)
__device__ __forceinline__ float pixel_lut(int32_t acc, int32_t b, int sh, const float* lut) {
  int v = (acc + b + (1 << (sh - 1))) >> sh;
  return lut[min(max(v, 0), 255)];
}

// ---- generic tile layer -------------------------------------------------------
template <int BN>
struct TileCfg {
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  static constexpr int NST = 4;
  static constexpr int SMEM = NST * STAGE_BYTES + 1024 + 256;
};

template <int BN, int EPI>
__global__ void __launch_bounds__(128)
    k_l8_tile(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const Args a) {
  using Cfg = TileCfg<BN>;
  constexpr int STAGES = Cfg::NST;
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
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
      const int tap = kb / a.kb_per_tap, cb = kb - tap * a.kb_per_tap;
      mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
      tc::tma_load_5d(sA + s * A_BYTES, &tmA, cb * KB, x0 + a.taps[tap][2], y0 + a.taps[tap][1],
                      t + a.taps[tap][0], g, &full[s]);
      tc::tma_load_2d(sB + s * Cfg::B_BYTES, &tmB, kb * KB, n0, &full[s]);
    }
  } else if (threadIdx.x == 32) {
    constexpr uint32_t idesc = tc::idesc_i8_s32(BM, BN);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      tc::fence_after_sync();
      const uint64_t ad = tc::smem_desc_sw128(smem_u32(sA + s * A_BYTES));
      const uint64_t bd = tc::smem_desc_sw128(smem_u32(sB + s * Cfg::B_BYTES));
#pragma unroll
      for (int k = 0; k < 4; ++k) tc::mma_i8(tmem, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
      tc::mma_commit(&empty[s]);
    }
    tc::mma_commit(accum);
  }
  __syncwarp();
  mbar_wait(accum, 0);
  tc::fence_after_sync();

  const int r = threadIdx.x;
  const int y = y0 + (r >> 4), x = x0 + (r & 15);
  const bool valid = y < a.Ht && x < a.Wt;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);

  if constexpr (EPI == SST_LT_EPI_STORE) {
    const size_t tok = (((size_t)g * a.out_T + t) * a.Ht + y) * a.Wt + x;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      float v[32];
      tc::tmem_ld32(trow + c, v);
      if (!valid) continue;
      uint4 res[2];
      const uint4* rp = nullptr;
      if (a.residual != nullptr) {
        const uint4* src = reinterpret_cast<const uint4*>(a.residual + tok * a.N + n0 + c);
        res[0] = __ldg(src);
        res[1] = __ldg(src + 1);
        rp = res;
      }
      uint4 o[2];
      epi_store32(v, a, n0 + c, rp, o);
      uint4* op = reinterpret_cast<uint4*>(a.out + tok * a.N + n0 + c);
      op[0] = o[0];
      op[1] = o[1];
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
        const int L = fsq_levels(i), hw = L / 2;
        int q = (__float_as_int(v[i]) + __ldg(a.bias + i)) >> a.shift;
        q = min(max(q, -hw), L - 1 - hw);
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
  } else {  // PIXELS: 192 columns = one frame's 8x8x3 patch
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
      if (a.pix_u8) {
        uint8_t* fr8 = reinterpret_cast<uint8_t*>(a.frames);
#pragma unroll
        for (int pr = 0; pr < 4; ++pr) {
          const int Y = y * 8 + half * 4 + pr;
          if (Y >= a.h) continue;
          const int X0 = x * 8;
          uint8_t* dst = fr8 + ((((size_t)g * 9 + f) * a.h + Y) * a.w + X0) * 3;
          const int npx = min(8, a.w - X0);
#pragma unroll
          for (int e = 0; e < 24; ++e) {
            if (e / 3 >= npx) continue;
            const int i = pr * 24 + e;
            const int r8 = (__float_as_int(v[i]) + __ldg(a.bias + n0 + half * 96 + i) +
                            (1 << (a.shift - 1))) >> a.shift;
            dst[e] = (uint8_t)min(max(r8, 0), 255);
          }
        }
        continue;
      }
#pragma unroll
      for (int i = 0; i < 96; ++i)
        v[i] = pixel(__float_as_int(v[i]), __ldg(a.bias + n0 + half * 96 + i), a.shift);
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

// ---- CTA-pair layer (cta_group::2) ---------------------------------------------
// The int8 port of learned.cu's k_lt_convpair: a cluster of 2 CTAs computes a
// unit of 256 tokens (16x16) x kNU output channels; CTA r owns x-half r of the
// tile (its own halo / token box and accumulator rows 128r..) and weight rows
// kNU/2 * r ..; the leader's single thread issues M=256 x N=kNU x K=32 MMAs.
// Causal (2,3,3) convs skip the temporal tap t-1 at t = 0 (it is all zero
// padding), so no MMA is spent on it.
namespace pc {
constexpr int TILE = 16, PITCH = 10, HROWS = 18;
constexpr int HALO_BYTES = PITCH * HROWS * 128;                   // 23040 (1x1: 8x16 box, 16384)
constexpr int HALO_STRIDE = (HALO_BYTES + 1023) / 1024 * 1024;    // 23552
// Epilogue warps per CTA: 8 (two per TMEM lane quarter) for the convs and
// the short-K GEMMs; 16 for the pixel layer, whose epilogue (requantise,
// pack, stage, scatter into frame rows) bounds it -- measured 200 -> 147 us
// for the P frames of 32 x 1080p GoPs, while the TMA-store GEMMs got slower
// with 16 (named-barrier halves of 8 warps)
template <bool kPix>
__host__ __device__ constexpr int epi_warps() { return kPix ? 16 : 8; }
template <bool kPix>
__host__ __device__ constexpr int pair_threads() { return 64 + 32 * epi_warps<kPix>(); }
}  // namespace pc

template <bool kHalo, bool kTma>
__host__ __device__ constexpr int pair_bstages() { return kHalo ? 8 : (kTma ? 6 : 8); }
template <bool kHalo>
__host__ __device__ constexpr int pair_hslots() { return kHalo ? 3 : 5; }
template <bool kHalo>
__host__ __device__ constexpr int pair_hstride() { return kHalo ? pc::HALO_STRIDE : 16384; }
template <bool kPix>
__host__ __device__ constexpr int pair_bbytes() { return (kPix ? 96 : 128) * 128; }
// TMA-store staging: [2 halves][128 rows][128 B]; pixel rows: 8 warps x 768 floats
template <bool kTma, bool kPix>
__host__ __device__ constexpr int pair_stage() {
  return kTma ? 2 * 16384 : (kPix ? pc::epi_warps<true>() * 3072 : 0);
}
template <bool kHalo, bool kTma, bool kPix = false>
__host__ __device__ constexpr int pair_smem() {
  return pair_hslots<kHalo>() * pair_hstride<kHalo>() + pair_bstages<kHalo, kTma>() * pair_bbytes<kPix>() +
         pair_stage<kTma, kPix>() + 1024 + 512;
}
static_assert(pair_smem<true, false>() <= 232448, "halo conv smem");
static_assert(pair_smem<false, true>() <= 232448, "1x1 conv smem");
static_assert(pair_smem<false, false, true>() <= 232448, "pixel conv smem");

__device__ __forceinline__ uint64_t halo_desc_pitch(uint32_t saddr, int pitch) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((pitch * 128) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <bool kHalo, bool kTma, bool kPix = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(pc::pair_threads<kPix>(), 1)
    k_l8_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmC, const Args a, int n_units, int n_blocks) {
  using namespace pc;
  constexpr int EPI_WARPS = epi_warps<kPix>();
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
  uint8_t* sStage = sB + BSTAGES * B_BYTES;
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
  __shared__ float pix_lut[kPix ? 256 : 1];
  if (kPix)
    for (int i = threadIdx.x; i < 256; i += blockDim.x) pix_lut[i] = __fdiv_rn((float)i, 255.0f);
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
  const int C = a.kb_per_tap * KB;
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
  // first halo block of a unit: at t = 0 the (2,3,3) conv's temporal tap t-1
  // reads only zero padding -- skip its loads and MMAs
  auto first_hi = [&](int t) { return (kHalo && t == 0) ? a.kb_per_tap : 0; };

  if (warp == 0) {
    if (lane == 0) {
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
            tc::tma_load_5d_pair(sH + hs * HALO_STRIDE, &tmA, cb * KB, x0 + 8 * (int)rank - 1,
                                 y0 - 1, t + kt - 1, g, &hfull[hs]);
          else
            tc::tma_load_5d_pair(sH + hs * HALO_STRIDE, &tmA, cb * KB, x0 + 8 * (int)rank, y0,
                                 t + a.taps[0][0], g, &hfull[hs]);
          for (int sp = 0; sp < kSpatial; ++sp, ++bc) {
            const int bs = bc % BSTAGES;
            if (bc >= BSTAGES) mbar_wait(&bempty[bs], ((bc / BSTAGES) - 1) & 1);
            if (leader) mbar_expect_tx(&bfull[bs], 2 * B_BYTES);
            tc::tma_load_2d_pair(sB + bs * B_BYTES, &tmB, (kt * kSpatial + sp) * C + cb * KB,
                                 nb * kNU + (int)rank * kBNH, &bfull[bs]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = tc::idesc_i8_s32(256, kNU);
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
            for (int k = 0; k < 4; ++k)
              tc::mma_i8_pair(acc, ad + 2 * k, bd + 2 * k, idesc, (hi != hi0 || sp | k) != 0);
            tc::mma_commit_pair(&bempty[bs]);
          }
          tc::mma_commit_pair(&hempty[hs]);
        }
        tc::mma_commit_pair(&afull[ab]);
      }
    }
  } else {
    // ---- epilogue (both CTAs): EPI_WARPS warps; warp w reads TMEM lanes
    // 32 (w % 4) .. +31 (its token rows) and column group cq = (w - 2) / 4 of
    // NCQ: 256 / NCQ columns of a 256-wide unit, or pixel rows 8 / NCQ .. of
    // a 192-wide pixel unit.  Column groups 0 .. NCQ/2 - 1 form TMA-store half 0.
    constexpr int NCQ = EPI_WARPS / 4;
    constexpr int HALF_WARPS = EPI_WARPS / 2;
    const int e = warp - 2;
    const int cq = e >> 2, q = warp & 3;
    const int half = e / HALF_WARPS;
    const int m = q * 32 + lane;
    const uint32_t aempty_leader = tc::mapa(smem_u32(&aempty[0]), 0);
    const bool issuer = kTma && (e % HALF_WARPS) == 0 && lane == 0;   // first warp of each half
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
        // 192 columns = 8 pixel rows x 8 pixels x 3 channels of the token
        constexpr int PR = 8 / NCQ;                  // pixel rows per warp
        constexpr int CW = PR * 24;                  // columns per warp
        const int prow0 = cq * PR;
        const uint32_t trp = tmem + ((uint32_t)(q * 32) << 16) + ab * 256 + cq * CW;
        float v[CW];
#pragma unroll
        for (int cc = 0; cc < CW / 16; ++cc) {
          float u16[16];
          tc::tmem_ld16(trp + cc * 16, u16);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[cc * 16 + i] = u16[i];
        }
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_cluster_relaxed(aempty_leader + ab * 8);
        const int f = a.frame_base + nb;
        const int nb0 = nb * kNU + cq * CW;
        const int4* bp4 = reinterpret_cast<const int4*>(a.bias + nb0);
        const int xs = x0 + 8 * (int)rank;
        if (a.pix_u8) {
          // uint8 q frames (sample value float(q / 255)): q in place of the
          // accumulator bits; the [0, 255] clamp happens in the saturating pack
          const int rnd = 1 << (a.shift - 1);
          auto qf = [&](int acc, int b) { return __int_as_float((acc + b + rnd) >> a.shift); };
#pragma unroll
          for (int i4 = 0; i4 < CW / 4; ++i4) {
            const int4 bb = __ldg(bp4 + i4);
            v[4 * i4 + 0] = qf(__float_as_int(v[4 * i4 + 0]), bb.x);
            v[4 * i4 + 1] = qf(__float_as_int(v[4 * i4 + 1]), bb.y);
            v[4 * i4 + 2] = qf(__float_as_int(v[4 * i4 + 2]), bb.z);
            v[4 * i4 + 3] = qf(__float_as_int(v[4 * i4 + 3]), bb.w);
          }
#define qv(i) __float_as_int(v[(i)])
          uint8_t* fr8 = reinterpret_cast<uint8_t*>(a.frames);
          const bool seg8 = (a.w * 3) % 16 == 0 && xs + 8 <= a.Wt && xs * 8 + 64 <= a.w;
          if (seg8) {
            uint8_t* srow = sStage + e * 768;                  // [4][192] bytes
#pragma unroll
            for (int pr = 0; pr < PR; ++pr) {
              uint32_t* s32 = reinterpret_cast<uint32_t*>(srow + (lane >> 3) * 192 + (lane & 7) * 24);
#pragma unroll
              for (int k = 0; k < 6; ++k)
                s32[k] = pack4_satu8(qv(pr * 24 + 4 * k), qv(pr * 24 + 4 * k + 1),
                                     qv(pr * 24 + 4 * k + 2), qv(pr * 24 + 4 * k + 3));
              __syncwarp();
              for (int i = lane; i < 48; i += 32) {
                const int r = i / 12, c16 = i - r * 12;
                const int yr = y0 + q * 4 + r;
                const int Y = yr * 8 + prow0 + pr;
                if (yr < a.Ht && Y < a.h)
                  reinterpret_cast<uint4*>(fr8 + ((((size_t)g * 9 + f) * a.h + Y) * a.w + xs * 8) * 3)[c16] =
                      reinterpret_cast<const uint4*>(srow + r * 192)[c16];
              }
              __syncwarp();
            }
            continue;
          }
          if (!valid) continue;
#pragma unroll
          for (int pr = 0; pr < PR; ++pr) {
            const int Y = y * 8 + prow0 + pr;
            if (Y >= a.h) continue;
            const int X0 = x * 8;
            uint8_t* dst = fr8 + ((((size_t)g * 9 + f) * a.h + Y) * a.w + X0) * 3;
            const int npx = min(8, a.w - X0);
#pragma unroll
            for (int k = 0; k < 24; ++k)
              if (k / 3 < npx) dst[k] = (uint8_t)min(max(qv(pr * 24 + k), 0), 255);
          }
#undef qv
          continue;
        }
#pragma unroll
        for (int i4 = 0; i4 < CW / 4; ++i4) {
          const int4 bb = __ldg(bp4 + i4);
          v[4 * i4 + 0] = pixel_lut(__float_as_int(v[4 * i4 + 0]), bb.x, a.shift, pix_lut);
          v[4 * i4 + 1] = pixel_lut(__float_as_int(v[4 * i4 + 1]), bb.y, a.shift, pix_lut);
          v[4 * i4 + 2] = pixel_lut(__float_as_int(v[4 * i4 + 2]), bb.z, a.shift, pix_lut);
          v[4 * i4 + 3] = pixel_lut(__float_as_int(v[4 * i4 + 3]), bb.w, a.shift, pix_lut);
        }
        const bool vec = (a.w & 3) == 0;
        const bool seg = vec && xs + 8 <= a.Wt && xs * 8 + 64 <= a.w;
        if (seg) {
          float* srow = reinterpret_cast<float*>(sStage) + e * 768;   // [4][192]
#pragma unroll
          for (int pr = 0; pr < PR; ++pr) {
            float4* s4 = reinterpret_cast<float4*>(srow + (lane >> 3) * 192 + (lane & 7) * 24);
#pragma unroll
            for (int e4 = 0; e4 < 6; ++e4)
              s4[e4] = make_float4(v[pr * 24 + 4 * e4], v[pr * 24 + 4 * e4 + 1],
                                   v[pr * 24 + 4 * e4 + 2], v[pr * 24 + 4 * e4 + 3]);
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 6; ++i) {
              const int idx = i * 32 + lane, r = idx / 48, c4 = idx - r * 48;
              const int yr = y0 + q * 4 + r;
              const int Y = yr * 8 + prow0 + pr;
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
        for (int pr = 0; pr < PR; ++pr) {
          const int Y = y * 8 + prow0 + pr;
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
      constexpr int CW = 256 / NCQ;                  // columns per warp
      const int n0 = nb * 256 + cq * CW;
      const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + ab * 256 + cq * CW;
      const size_t tok = (((size_t)g * a.out_T + t) * a.Ht + y) * a.Wt + x;
      if constexpr (kTma) {
        // short-K GEMM epilogue: the row's residual bytes up front, the wait
        // for the previous unit's TMA store deferred to the first write
        uint8_t* stage = sStage + half * 16384;
        const int co = (cq * CW) & 127;              // column offset inside the half
        uint4 res[CW / 16];
        const bool has_res = valid && a.residual != nullptr;
        if (has_res) {
          const uint4* rp = reinterpret_cast<const uint4*>(a.residual + tok * a.N + n0);
#pragma unroll
          for (int i = 0; i < CW / 16; ++i) res[i] = __ldg(rp + i);
        }
#pragma unroll
        for (int c = 0; c < CW; c += 32) {
          float v[32];
          tc::tmem_ld32(trow + c, v);
          if (c + 32 == CW) {
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive_cluster_relaxed(aempty_leader + ab * 8);
          }
          uint4 o[2];
          epi_store32(v, a, n0 + c, has_res ? &res[c >> 4] : nullptr, o);
          if (c == 0) {
            if (issuer) tma_store_wait_read();
            named_bar(1 + half, 32 * HALF_WARPS);
          }
          const int j0 = (co + c) >> 4;
#pragma unroll
          for (int qq = 0; qq < 2; ++qq)
            *reinterpret_cast<uint4*>(stage + m * 128 + (((j0 + qq) ^ (m & 7)) << 4)) = o[qq];
        }
        fence_proxy_async_smem();
        named_bar(1 + half, 32 * HALF_WARPS);
        if (issuer) {
          tc::tma_store_5d(&tmC, stage, nb * 256 + half * 128, x0 + 8 * (int)rank, y0, t, g);
          tma_store_commit();
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < CW; c += 32) {
          float v[32];
          tc::tmem_ld32(trow + c, v);
          if (c + 32 == CW) {
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive_cluster_relaxed(aempty_leader + ab * 8);
          }
          if (!valid) continue;
          uint4 res[2];
          const uint4* rp = nullptr;
          if (a.residual != nullptr) {
            const uint4* src = reinterpret_cast<const uint4*>(a.residual + tok * a.N + n0 + c);
            res[0] = __ldg(src);
            res[1] = __ldg(src + 1);
            rp = res;
          }
          uint4 o[2];
          epi_store32(v, a, n0 + c, rp, o);
          uint4* op = reinterpret_cast<uint4*>(a.out + tok * a.N + n0 + c);
          op[0] = o[0];
          op[1] = o[1];
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

// ---- causal window attention, integer softmax --------------------------------
// One CTA = one (GoP, 8x8 window, 128-dim head): 128 query rows (2 latent
// frames x 64 tokens) against the same 128 keys.
//   S = Q K^T   kind::i8 (s8 x s8), M=128 N=128 K=128 -> TMEM columns 0..127
//   softmax     thread q, two passes over its TMEM row: m = max allowed S,
//               then e = EXP[min((m - S) >> sh, 255)] (allowed: valid token of
//               a frame <= the query's), l = sum e, P = e (uint8) -> smem (over Q)
//   O = P V     kind::i8 (u8 x s8), M=128 N=128 K=128 -> the same TMEM columns
//               (every S value is in registers / smem by then); V is the B
//               operand in MN-major form: its rows are the keys exactly as
//               loaded, no transposed scatter
//   out         clamp(floor((2 O + l) / (2 l)), -127, 127) -> int8 (division by
//               a float reciprocal, corrected to the exact integer floor)
// 128 TMEM columns and ~50 KB of smem per CTA: four CTAs share an SM.
constexpr int AT_WIN = 8, AT_HD = 128;
constexpr int AT_SMEM = 3 * 16384 + 1024 + 64 + 128 * 4 + 256;

__device__ __forceinline__ int floor_div_pos(int n, int d, float rcp) {
  int q = __float2int_rd((float)n * rcp);       // |n| < 2^24: within one of the floor
  int r = n - q * d;
  if (r < 0) { --q; r += d; }
  if (r >= d) ++q;
  return q;
}

__global__ void __launch_bounds__(128, 4)
    k_l8_attn(const int8_t* __restrict__ qkv, int G, int Ht, int Wt, int D, int shift,
              const uint8_t* __restrict__ exp_lut, int8_t* __restrict__ out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;                 // [128 q][128 d]  A of S; then P [128 q][128 k], A of O
  uint8_t* sK = smem + 16384;         // [128 k][128 d]  B of S (K-major)
  uint8_t* sV = smem + 32768;         // [128 k][128 d]  B of O (MN-major: d contiguous)
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 49152);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2);
  int* kval = reinterpret_cast<int*>(smem + 49152 + 64);
  uint8_t* lut = smem + 49152 + 64 + 512;

  const int wins_x = ceil_div(Wt, AT_WIN);
  const int wy = blockIdx.x / wins_x, wx = blockIdx.x - wy * wins_x;
  const int head = blockIdx.y, g = blockIdx.z;
  const int t = threadIdx.x, warp = t >> 5;
  const int ft = t >> 6, lt = t & 63;
  const int y = wy * AT_WIN + (lt >> 3), x = wx * AT_WIN + (lt & 7);
  const bool valid = y < Ht && x < Wt;
  const size_t tok = (((size_t)g * 2 + ft) * Ht + y) * Wt + x;

  if (t == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 128);
  lut[t] = exp_lut[t];
  lut[t + 128] = exp_lut[t + 128];
  kval[t] = valid;
  {
    const uint4* base = reinterpret_cast<const uint4*>(qkv + tok * 3 * D + head * AT_HD);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint4 q4 = make_uint4(0, 0, 0, 0), k4 = q4, v4 = q4;
      if (valid) {
        q4 = __ldg(base + j);
        k4 = __ldg(base + D / 16 + j);
        v4 = __ldg(base + 2 * D / 16 + j);
      }
      const int off = t * 128 + ((j ^ (t & 7)) << 4);
      *reinterpret_cast<uint4*>(sQ + off) = q4;
      *reinterpret_cast<uint4*>(sK + off) = k4;
      *reinterpret_cast<uint4*>(sV + off) = v4;
    }
  }
  fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (t == 0) {
    constexpr uint32_t id1 = tc::idesc_i8_s32(128, 128, true, true);
    const uint64_t ad = tc::smem_desc_sw128(smem_u32(sQ));
    const uint64_t bd = tc::smem_desc_sw128(smem_u32(sK));
#pragma unroll
    for (int k = 0; k < 4; ++k) tc::mma_i8(tmem, ad + 2 * k, bd + 2 * k, id1, k);
    tc::mma_commit(&bar[0]);
  }
  mbar_wait(&bar[0], 0);
  tc::fence_after_sync();

  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  const int nk = (ft + 1) * 64;       // causal: keys of frames <= ft
  int m = INT_MIN;
#pragma unroll 1
  for (int c = 0; c < nk; c += 32) {
    float v[32];
    tc::tmem_ld32(trow + c, v);
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (kval[c + i]) m = max(m, __float_as_int(v[i]));
  }
  int l = 0;
#pragma unroll 1
  for (int c = 0; c < 128; c += 32) {
    int e[32];
    if (c < nk) {
      float v[32];
      tc::tmem_ld32(trow + c, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        e[i] = kval[c + i] ? (int)lut[min((m - __float_as_int(v[i])) >> shift, 255)] : 0;
        l += e[i];
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) e[i] = 0;
    }
    // P row t, keys c..c+31 = 16-byte chunks c/16, c/16+1 (over Q: the S MMA has retired)
#pragma unroll
    for (int qq = 0; qq < 2; ++qq) {
      const int j = (c >> 4) + qq;
      const int* ee = e + 16 * qq;
      *reinterpret_cast<uint4*>(sQ + t * 128 + ((j ^ (t & 7)) << 4)) =
          make_uint4(pack4(ee[0], ee[1], ee[2], ee[3]), pack4(ee[4], ee[5], ee[6], ee[7]),
                     pack4(ee[8], ee[9], ee[10], ee[11]), pack4(ee[12], ee[13], ee[14], ee[15]));
    }
  }
  fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();                    // every S value read: O may overwrite its columns
  tc::fence_after_sync();
  if (t == 0) {
    // P unsigned, V signed and MN-major (bit 16): a K step of 32 keys is 32
    // rows = 4 swizzle atoms = 4096 bytes
    constexpr uint32_t id2 = tc::idesc_i8_s32(128, 128, false, true) | (1u << 16);
    const uint64_t ad = tc::smem_desc_sw128(smem_u32(sQ));
    const uint64_t bd = tc::smem_desc_sw128(smem_u32(sV));
#pragma unroll
    for (int k = 0; k < 4; ++k) tc::mma_i8(tmem, ad + 2 * k, bd + 256 * k, id2, k);
    tc::mma_commit(&bar[1]);
  }
  mbar_wait(&bar[1], 0);
  tc::fence_after_sync();
  const int l2 = 2 * l;
  const float rcp = 1.0f / (float)l2;
#pragma unroll 1
  for (int c = 0; c < 128; c += 32) {
    float v[32];
    tc::tmem_ld32(trow + c, v);
    if (!valid) continue;
    int o[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int q = floor_div_pos(2 * __float_as_int(v[i]) + l, l2, rcp);
      o[i] = min(max(q, -127), 127);
    }
    uint4* op = reinterpret_cast<uint4*>(out + tok * D + head * AT_HD + c);
#pragma unroll
    for (int qq = 0; qq < 2; ++qq)
      op[qq] = make_uint4(pack4(o[qq * 16 + 0], o[qq * 16 + 1], o[qq * 16 + 2], o[qq * 16 + 3]),
                          pack4(o[qq * 16 + 4], o[qq * 16 + 5], o[qq * 16 + 6], o[qq * 16 + 7]),
                          pack4(o[qq * 16 + 8], o[qq * 16 + 9], o[qq * 16 + 10], o[qq * 16 + 11]),
                          pack4(o[qq * 16 + 12], o[qq * 16 + 13], o[qq * 16 + 14], o[qq * 16 + 15]));
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 128);
}

// ---- global causal attention (full-frame keys), integer softmax --------------
// One CTA = one (GoP, latent frame t, 128-query tile, 128-dim head).  The
// query attends every token of frames <= t (2 x H' x W' keys at t = 1), so the
// keys stream through shared memory in tiles of 128 in two passes: pass 1
// finds the row max (S = Q K^T per tile on tcgen05), pass 2 recomputes each
// tile's S, forms P = EXP[min((max - S) >> sh, 255)] and accumulates O += P V
// in TMEM (int32, exact in any order) -- the same arithmetic as the windowed
// kernel over all keys, so the result is still bit-exact to the oracle.
constexpr int AG_SMEM = 4 * 16384 + 1024 + 64 + 256;

__global__ void __launch_bounds__(128, 2)
    k_l8_attn_global(const int8_t* __restrict__ qkv, int G, int n, int D, int shift,
                     const uint8_t* __restrict__ exp_lut, int8_t* __restrict__ out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;                 // [128 q][128 d]      A of S
  uint8_t* sK = smem + 16384;         // [128 k][128 d]      B of S (K-major)
  uint8_t* sV = smem + 32768;         // [128 k][128 d]      B of O (MN-major)
  uint8_t* sP = smem + 49152;         // [128 q][128 k] u8   A of O
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2);
  uint8_t* lut = smem + 65536 + 64;

  const int head = blockIdx.y;
  const int g = blockIdx.z >> 1, t = blockIdx.z & 1;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int qi = blockIdx.x * 128 + tid;
  const bool valid_q = qi < n;
  const size_t tok_q = ((size_t)g * 2 + t) * n + qi;
  const int nkeys = (t + 1) * n;
  const int ntiles = (nkeys + 127) / 128;

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 256);
  lut[tid] = exp_lut[tid];
  lut[tid + 128] = exp_lut[tid + 128];
  {
    const uint4* qb = reinterpret_cast<const uint4*>(qkv + tok_q * 3 * D + head * AT_HD);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      *reinterpret_cast<uint4*>(sQ + tid * 128 + ((j ^ (tid & 7)) << 4)) =
          valid_q ? __ldg(qb + j) : make_uint4(0, 0, 0, 0);
  }
  auto load_kv = [&](int kt, bool with_v) {
    const int k = kt * 128 + tid;
    const bool vk = k < nkeys;
    const int tt = vk ? k / n : 0, pos = vk ? k - tt * n : 0;
    const uint4* kb = reinterpret_cast<const uint4*>(
        qkv + (((size_t)g * 2 + tt) * n + pos) * 3 * D + D + head * AT_HD);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int off = tid * 128 + ((j ^ (tid & 7)) << 4);
      *reinterpret_cast<uint4*>(sK + off) = vk ? __ldg(kb + j) : make_uint4(0, 0, 0, 0);
      if (with_v)
        *reinterpret_cast<uint4*>(sV + off) = vk ? __ldg(kb + D / 16 + j) : make_uint4(0, 0, 0, 0);
    }
    fence_proxy_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
  };
  fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  constexpr uint32_t id1 = tc::idesc_i8_s32(128, 128, true, true);
  constexpr uint32_t id2 = tc::idesc_i8_s32(128, 128, false, true) | (1u << 16);
  uint32_t ph0 = 0, ph1 = 0;
  auto mma_s = [&]() {
    if (tid == 0) {
      const uint64_t ad = tc::smem_desc_sw128(smem_u32(sQ));
      const uint64_t bd = tc::smem_desc_sw128(smem_u32(sK));
#pragma unroll
      for (int k = 0; k < 4; ++k) tc::mma_i8(tmem, ad + 2 * k, bd + 2 * k, id1, k);
      tc::mma_commit(&bar[0]);
    }
    mbar_wait(&bar[0], ph0);
    ph0 ^= 1;
    tc::fence_after_sync();
  };

  // ---- pass 1: row max over all allowed keys ----
  int m = INT_MIN;
  for (int kt = 0; kt < ntiles; ++kt) {
    load_kv(kt, false);
    mma_s();
#pragma unroll 1
    for (int c = 0; c < 128; c += 32) {
      float v[32];
      tc::tmem_ld32(trow + c, v);
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (kt * 128 + c + i < nkeys) m = max(m, __float_as_int(v[i]));
    }
    tc::fence_before_sync();
    __syncthreads();                  // S read by every thread, sK free
  }
  // ---- pass 2: P = EXP[...], l = sum P, O += P V ----
  int l = 0;
  for (int kt = 0; kt < ntiles; ++kt) {
    load_kv(kt, true);
    mma_s();
#pragma unroll 1
    for (int c = 0; c < 128; c += 32) {
      float v[32];
      tc::tmem_ld32(trow + c, v);
      int e[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const bool ok = valid_q && kt * 128 + c + i < nkeys;
        e[i] = ok ? (int)lut[min((m - __float_as_int(v[i])) >> shift, 255)] : 0;
        l += e[i];
      }
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
        const int j = (c >> 4) + qq;
        const int* ee = e + 16 * qq;
        *reinterpret_cast<uint4*>(sP + tid * 128 + ((j ^ (tid & 7)) << 4)) =
            make_uint4(pack4(ee[0], ee[1], ee[2], ee[3]), pack4(ee[4], ee[5], ee[6], ee[7]),
                       pack4(ee[8], ee[9], ee[10], ee[11]), pack4(ee[12], ee[13], ee[14], ee[15]));
      }
    }
    fence_proxy_async_smem();
    tc::fence_before_sync();
    __syncthreads();                  // P complete, S read: O may accumulate
    tc::fence_after_sync();
    if (tid == 0) {
      const uint64_t ad = tc::smem_desc_sw128(smem_u32(sP));
      const uint64_t bd = tc::smem_desc_sw128(smem_u32(sV));
#pragma unroll
      for (int k = 0; k < 4; ++k) tc::mma_i8(tmem + 128, ad + 2 * k, bd + 256 * k, id2, (kt | k) != 0);
      tc::mma_commit(&bar[1]);
    }
    mbar_wait(&bar[1], ph1);          // sP / sV / S free for the next tile
    ph1 ^= 1;
    tc::fence_after_sync();
  }
  const int l2 = 2 * max(l, 1);
  const float rcp = 1.0f / (float)l2;
#pragma unroll 1
  for (int c = 0; c < 128; c += 32) {
    float v[32];
    tc::tmem_ld32(trow + 128 + c, v);
    if (!valid_q) continue;
    int o[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int q = floor_div_pos(2 * __float_as_int(v[i]) + l, l2, rcp);
      o[i] = min(max(q, -127), 127);
    }
    uint4* op = reinterpret_cast<uint4*>(out + tok_q * D + head * AT_HD + c);
#pragma unroll
    for (int qq = 0; qq < 2; ++qq)
      op[qq] = make_uint4(pack4(o[qq * 16 + 0], o[qq * 16 + 1], o[qq * 16 + 2], o[qq * 16 + 3]),
                          pack4(o[qq * 16 + 4], o[qq * 16 + 5], o[qq * 16 + 6], o[qq * 16 + 7]),
                          pack4(o[qq * 16 + 8], o[qq * 16 + 9], o[qq * 16 + 10], o[qq * 16 + 11]),
                          pack4(o[qq * 16 + 12], o[qq * 16 + 13], o[qq * 16 + 14], o[qq * 16 + 15]));
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}

// ---- global causal attention, TMA-pipelined (default) ----------------------------
// The same arithmetic as k_l8_attn_global, with the key / value tiles brought
// in by TMA two jobs ahead instead of loaded synchronously by every thread:
// the 2 x ntiles jobs (pass 1: K tiles for the row max; pass 2: K + V tiles for
// P and O += P V) rotate through two smem stages, and thread 0 re-arms a stage
// with job j + 2 as soon as job j's MMAs have consumed it.  The tiles come
// straight from the [tokens][3 D] qkv rows through a 2-D tensor map with the
// 128-byte swizzle the UMMA descriptors expect (K-major Q / K, MN-major V);
// rows past the allowed keys are masked in the softmax as before.  The integer
// softmax needs the exact row max before any P, so the two passes stay.
constexpr int AG2_SMEM = 6 * 16384 + 1024 + 64 + 256;

__global__ void __launch_bounds__(128, 2)
    k_l8_attn_global_tma(const __grid_constant__ CUtensorMap tq, int G, int n, int D, int shift,
                         const uint8_t* __restrict__ exp_lut, int8_t* __restrict__ out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;                         // [128 q][128 d]            A of S
  uint8_t* sKV = smem + 16384;                // 2 stages x {K, V} [128][128]
  uint8_t* sP = smem + 5 * 16384;             // [128 q][128 k] u8         A of O
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 6 * 16384);   // full0 full1 q s o
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 5);
  uint8_t* lut = smem + 6 * 16384 + 64;

  const int head = blockIdx.y;
  const int g = blockIdx.z >> 1, t = blockIdx.z & 1;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int qi = blockIdx.x * 128 + tid;
  const bool valid_q = qi < n;
  const size_t tok_q = ((size_t)g * 2 + t) * n + qi;
  const int nkeys = (t + 1) * n;
  const int ntiles = (nkeys + 127) / 128;
  const int njobs = 2 * ntiles;
  const int row0 = g * 2 * n;                 // first token row of this GoP
  const int xk = D + head * AT_HD, xv = 2 * D + head * AT_HD;

  auto issue = [&](int j) {                   // job j -> stage j & 1
    const int st = j & 1;
    const bool p2 = j >= ntiles;
    const int kt = p2 ? j - ntiles : j;
    uint8_t* dk = sKV + st * 32768;
    mbar_expect_tx(&bar[st], p2 ? 32768u : 16384u);
    tc::tma_load_2d(dk, &tq, xk, row0 + kt * 128, &bar[st]);
    if (p2) tc::tma_load_2d(dk + 16384, &tq, xv, row0 + kt * 128, &bar[st]);
  };
  if (tid == 0) {
    for (int i = 0; i < 5; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
    tc::prefetch_tmap(&tq);
    mbar_expect_tx(&bar[2], 16384u);
    tc::tma_load_2d(sQ, &tq, head * AT_HD, row0 + t * n + blockIdx.x * 128, &bar[2]);
    issue(0);
    if (njobs > 1) issue(1);
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 256);
  lut[tid] = exp_lut[tid];
  lut[tid + 128] = exp_lut[tid + 128];
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  constexpr uint32_t id1 = tc::idesc_i8_s32(128, 128, true, true);
  constexpr uint32_t id2 = tc::idesc_i8_s32(128, 128, false, true) | (1u << 16);
  if (tid == 0) mbar_wait(&bar[2], 0);
  uint32_t ph_s = 0, ph_o = 0;
  int m = INT_MIN;
  uint32_t lsum = 0;
  const int lim = (256 << shift) - 1;
  for (int j = 0; j < njobs; ++j) {
    const int st = j & 1;
    const bool p2 = j >= ntiles;
    const int kt = p2 ? j - ntiles : j;
    uint8_t* sK = sKV + st * 32768;
    if (tid == 0) {
      mbar_wait(&bar[st], (j >> 1) & 1);
      const uint64_t ad = tc::smem_desc_sw128(smem_u32(sQ));
      const uint64_t bd = tc::smem_desc_sw128(smem_u32(sK));
#pragma unroll
      for (int k = 0; k < 4; ++k) tc::mma_i8(tmem, ad + 2 * k, bd + 2 * k, id1, k);
      tc::mma_commit(&bar[3]);
    }
    mbar_wait(&bar[3], ph_s);
    ph_s ^= 1;
    tc::fence_after_sync();
    if (!p2) {
      // pass 1: row max over all allowed keys
      const bool full = (kt + 1) * 128 <= nkeys;   // every key of the tile allowed
#pragma unroll 1
      for (int c = 0; c < 128; c += 32) {
        float v[32];
        tc::tmem_ld32(trow + c, v);
        if (full) {
          int m2[4] = {m, m, m, m};
#pragma unroll
          for (int i = 0; i < 32; ++i) m2[i & 3] = max(m2[i & 3], __float_as_int(v[i]));
          m = max(max(m2[0], m2[1]), max(m2[2], m2[3]));
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (kt * 128 + c + i < nkeys) m = max(m, __float_as_int(v[i]));
        }
      }
      tc::fence_before_sync();
      __syncthreads();                        // S read: TMEM S and stage st are free
      if (tid == 0 && j + 2 < njobs) issue(j + 2);
      continue;
    }
    // pass 2: P = EXP[...], l = sum P, O += P V
    const bool full = valid_q && (kt + 1) * 128 <= nkeys;
#pragma unroll 1
    for (int c = 0; c < 128; c += 32) {
      float v[32];
      tc::tmem_ld32(trow + c, v);
      int e[32];
      if (full) {
        // (m - S) >= 0 for every allowed key: min(m - S, lim) >> sh is
        // min((m - S) >> sh, 255) in one add-min plus a shift
#pragma unroll
        for (int i = 0; i < 32; ++i)
          e[i] = (int)lut[(uint32_t)min(m - __float_as_int(v[i]), lim) >> shift];
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const bool ok = valid_q && kt * 128 + c + i < nkeys;
          e[i] = ok ? (int)lut[min((m - __float_as_int(v[i])) >> shift, 255)] : 0;
        }
      }
      uint32_t w[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        w[k] = pack4_satu8(e[4 * k], e[4 * k + 1], e[4 * k + 2], e[4 * k + 3]);
        lsum = __dp4a(w[k], 0x01010101u, lsum);      // l += the four P bytes
      }
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
        const int jj = (c >> 4) + qq;
        *reinterpret_cast<uint4*>(sP + tid * 128 + ((jj ^ (tid & 7)) << 4)) =
            make_uint4(w[4 * qq], w[4 * qq + 1], w[4 * qq + 2], w[4 * qq + 3]);
      }
    }
    fence_proxy_async_smem();
    tc::fence_before_sync();
    __syncthreads();                          // P complete, S read: O may accumulate
    tc::fence_after_sync();
    if (tid == 0) {
      const uint64_t ad = tc::smem_desc_sw128(smem_u32(sP));
      const uint64_t bd = tc::smem_desc_sw128(smem_u32(sK + 16384));
#pragma unroll
      for (int k = 0; k < 4; ++k) tc::mma_i8(tmem + 128, ad + 2 * k, bd + 256 * k, id2, (kt | k) != 0);
      tc::mma_commit(&bar[4]);
    }
    mbar_wait(&bar[4], ph_o);                 // sP, stage st and TMEM S free
    ph_o ^= 1;
    tc::fence_after_sync();
    if (tid == 0 && j + 2 < njobs) issue(j + 2);
  }
  const int l = (int)lsum;
  const int l2 = 2 * max(l, 1);
  const float rcp = 1.0f / (float)l2;
#pragma unroll 1
  for (int c = 0; c < 128; c += 32) {
    float v[32];
    tc::tmem_ld32(trow + 128 + c, v);
    if (!valid_q) continue;
    int o[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int q = floor_div_pos(2 * __float_as_int(v[i]) + l, l2, rcp);
      o[i] = min(max(q, -127), 127);
    }
    uint4* op = reinterpret_cast<uint4*>(out + tok_q * D + head * AT_HD + c);
#pragma unroll
    for (int qq = 0; qq < 2; ++qq)
      op[qq] = make_uint4(pack4(o[qq * 16 + 0], o[qq * 16 + 1], o[qq * 16 + 2], o[qq * 16 + 3]),
                          pack4(o[qq * 16 + 4], o[qq * 16 + 5], o[qq * 16 + 6], o[qq * 16 + 7]),
                          pack4(o[qq * 16 + 8], o[qq * 16 + 9], o[qq * 16 + 10], o[qq * 16 + 11]),
                          pack4(o[qq * 16 + 12], o[qq * 16 + 13], o[qq * 16 + 14], o[qq * 16 + 15]));
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}

// ---- patchify -------------------------------------------------------------------
template <int S>
__global__ void k_l8_patchify(const float* __restrict__ src, int G, int H, int W, int h, int w,
                              int Ht, int Wt, int8_t* __restrict__ pI, int8_t* __restrict__ pP) {
  const int PW = Wt * 8;
  const int X = blockIdx.x * blockDim.x + threadIdx.x;
  if (X >= PW) return;
  const int Y = blockIdx.y;
  const int f = (int)(blockIdx.z % 9);
  const int g = (int)(blockIdx.z / 9);
  const int xc = min(X, w - 1), yc = min(Y, h - 1);  // np.pad(mode="edge") of the working frame
  const float* fr = src + ((int64_t)g * 9 + f) * (int64_t)H * W * 3;
  int8_t px[3];
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    float v;
    if (S == 1) {
      v = __ldg(fr + ((int64_t)yc * W + xc) * 3 + ch);
    } else {
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
      v = __double2float_rn(acc / (double)(S * S));
    }
    px[ch] = (int8_t)((int)rint(__dmul_rn((double)v, 255.0)) - 128);
  }
  const int ty = Y >> 3, py = Y & 7, tx = X >> 3, pxl = X & 7;
  int8_t* dst;
  if (f == 0) {
    int8_t* tokb = pI + ((int64_t)(g * Ht + ty) * Wt + tx) * 256;
    dst = tokb + (py * 8 + pxl) * 3;
    if (py == 7 && pxl < 4)               // zero the 64 padding channels 192..255
      reinterpret_cast<uint4*>(tokb + 192)[pxl] = make_uint4(0, 0, 0, 0);
  } else {
    dst = pP + ((int64_t)(g * Ht + ty) * Wt + tx) * 1536 + (((f - 1) * 8 + py) * 8 + pxl) * 3;
  }
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) dst[ch] = px[ch];
}

// ---- patchify through the integer 3-D Haar front end -------------------------------
// One CTA per (GoP, token row, 8 tokens): 64 x 8 threads, one pixel column of
// the 8-row band each.  Each thread loads its pixel in all nine frames,
// quantises it, runs the three temporal levels over the P frames in
// registers and stores the frame slots straight into the OUTPUT layout held
// in shared memory (I [8][256], P [8][1536]); the spatial levels then run
// line by line in place (one thread per 8-, 4- or 2-long row / column of a
// (frame slot, token, channel) plane), and the band leaves as two contiguous
// 16-byte-vector runs.  Every coefficient stays in [-128, 127].
constexpr int kHaarTok = 8;                 // tokens per CTA
constexpr int kHaarThreads = kHaarTok * 8 * 8;

template <int M>
__device__ __forceinline__ void haar_line(int8_t* p, int stride) {
  int v[M];
#pragma unroll
  for (int j = 0; j < M; ++j) v[j] = p[j * stride];
#pragma unroll
  for (int j = 0; j < M / 2; ++j) {
    p[j * stride] = (int8_t)((v[2 * j] + v[2 * j + 1]) >> 1);
    p[(M / 2 + j) * stride] = (int8_t)((v[2 * j] - v[2 * j + 1]) >> 1);
  }
}

template <int M>
__device__ __forceinline__ void haar_regs(int (&v)[8]) {
  int t[M];
#pragma unroll
  for (int j = 0; j < M / 2; ++j) {
    t[j] = (v[2 * j] + v[2 * j + 1]) >> 1;
    t[M / 2 + j] = (v[2 * j] - v[2 * j + 1]) >> 1;
  }
#pragma unroll
  for (int j = 0; j < M; ++j) v[j] = t[j];
}

// spatial level M over every (frame slot, token, channel) plane of the band
template <int M>
__device__ __forceinline__ void haar_spatial(int8_t* sI, int8_t* sP, int tid) {
  constexpr int kPlanes = 9 * kHaarTok * 3;
  // horizontal: row r < M of each plane, stride 3 (channel-interleaved)
  for (int u = tid; u < kPlanes * M; u += kHaarThreads) {
    const int r = u % M, pl = u / M;
    const int ch = pl % 3, tok = (pl / 3) % kHaarTok, f = pl / (3 * kHaarTok);
    int8_t* base = f == 0 ? sI + tok * 256 : sP + tok * 1536 + (f - 1) * 192;
    haar_line<M>(base + r * 24 + ch, 3);
  }
  __syncthreads();
  for (int u = tid; u < kPlanes * M; u += kHaarThreads) {       // vertical: column c < M
    const int c = u % M, pl = u / M;
    const int ch = pl % 3, tok = (pl / 3) % kHaarTok, f = pl / (3 * kHaarTok);
    int8_t* base = f == 0 ? sI + tok * 256 : sP + tok * 1536 + (f - 1) * 192;
    haar_line<M>(base + c * 3 + ch, 24);
  }
  __syncthreads();
}

template <int S, bool kHaar>
__global__ void __launch_bounds__(kHaarThreads, 2)
    k_l8_patchify_band(const float* __restrict__ src, int H, int W, int h, int w, int Ht, int Wt,
                       int8_t* __restrict__ pI, int8_t* __restrict__ pP) {
  __shared__ __align__(16) int8_t sI[kHaarTok * 256];
  __shared__ __align__(16) int8_t sP[kHaarTok * 1536];
  const int tid = threadIdx.x;
  const int lx = tid & 63, py = tid >> 6;          // 64 pixel columns x 8 rows
  const int tx0 = blockIdx.x * kHaarTok, ty = blockIdx.y, g = blockIdx.z;
  const int X = tx0 * 8 + lx, Y = ty * 8 + py;
  const int tok = lx >> 3, pxl = lx & 7;
  const int xc = min(X, w - 1), yc = min(Y, h - 1);  // np.pad(mode="edge")
  int q[3][8];                                      // P frames 1..8 per channel
  int qi[3];
  const bool live = X < Wt * 8;
#pragma unroll
  for (int f = 0; f < 9; ++f) {
    const float* fr = src + ((int64_t)g * 9 + f) * (int64_t)H * W * 3;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      int val = 0;
      if (live) {
        float v;
        if (S == 1) {
          v = __ldg(fr + ((int64_t)yc * W + xc) * 3 + ch);
        } else {
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
          v = __double2float_rn(acc / (double)(S * S));
        }
        val = (int)rint(__dmul_rn((double)v, 255.0)) - 128;
      }
      if (f == 0) qi[ch] = val;
      else q[ch][f - 1] = val;
    }
  }
  if (kHaar) {
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {                // temporal levels 8 -> 4 -> 2
      haar_regs<8>(q[ch]);
      haar_regs<4>(q[ch]);
      haar_regs<2>(q[ch]);
    }
  }
  const int po = (py * 8 + pxl) * 3;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    sI[tok * 256 + po + ch] = (int8_t)qi[ch];
#pragma unroll
    for (int f = 0; f < 8; ++f) sP[tok * 1536 + f * 192 + po + ch] = (int8_t)q[ch][f];
  }
  if (py == 7 && pxl < 4)                           // channels 192..255 of I are zero
    reinterpret_cast<uint4*>(sI + tok * 256 + 192)[pxl] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  if (kHaar) {
    haar_spatial<8>(sI, sP, tid);
    haar_spatial<4>(sI, sP, tid);
    haar_spatial<2>(sI, sP, tid);
  }
  const int ntok = min(kHaarTok, Wt - tx0);
  const int64_t t0 = (int64_t)(g * Ht + ty) * Wt + tx0;
  uint4* dI = reinterpret_cast<uint4*>(pI + t0 * 256);
  uint4* dP = reinterpret_cast<uint4*>(pP + t0 * 1536);
  const uint4* s4I = reinterpret_cast<const uint4*>(sI);
  const uint4* s4P = reinterpret_cast<const uint4*>(sP);
  for (int i = tid; i < ntok * 16; i += kHaarThreads) dI[i] = s4I[i];
  for (int i = tid; i < ntok * 96; i += kHaarThreads) dP[i] = s4P[i];
}

// ---- launchers ----------------------------------------------------------------------
static void fill_args(Args& a, const SstConvDesc* d, int tile_x, int tile_y) {
  memset(&a, 0, sizeof(a));
  a.Ht = d->Ht; a.Wt = d->Wt;
  a.tiles_x = ceil_div(d->Wt, tile_x);
  a.tiles_y = ceil_div(d->Ht, tile_y);
  a.t_lo = d->t_lo; a.t_cnt = d->t_cnt;
  a.n_taps = d->n_taps;
  for (int i = 0; i < d->n_taps; ++i)
    for (int j = 0; j < 3; ++j) a.taps[i][j] = (signed char)d->taps[i][j];
  a.kb_per_tap = d->in_C / KB;
  a.N = d->N;
  a.out_T = d->out_T;
  a.bias = d->bias_i32;
  a.shift = d->shift;
  a.act = d->act;
  a.lut = d->act_lut;
  a.residual = static_cast<const int8_t*>(d->residual);
  a.out = static_cast<int8_t*>(d->out);
  a.codes = d->codes; a.idx = d->idx; a.mask = d->mask;
  a.frames = d->frames; a.h = d->h; a.w = d->w; a.frame_base = d->frame_base;
  a.pix_u8 = d->epi == SST_LT_EPI_PIXELS_U8;
}

template <int BN, int EPI>
static int launch_tile(const SstConvDesc* d, cudaStream_t st) {
  using Cfg = TileCfg<BN>;
  if (d->N % BN != 0) return SST_ERR_ARG;
  CUtensorMap tmA, tmB;
  memset(&tmA, 0, sizeof(tmA));
  memset(&tmB, 0, sizeof(tmB));
  const uint64_t adims[5] = {(uint64_t)d->in_C, (uint64_t)d->in_W, (uint64_t)d->in_H,
                             (uint64_t)d->in_T, (uint64_t)d->G};
  if (!make_tmap_u8_5d(&tmA, d->in, adims, BOX_X, BOX_Y)) return SST_ERR_ARG;
  if (!make_tmap_u8_2d(&tmB, d->weight, (uint64_t)d->K, (uint64_t)d->N, BN)) return SST_ERR_ARG;
  Args a;
  fill_args(a, d, BOX_X, BOX_Y);
  const int64_t mt = (int64_t)d->G * d->t_cnt * a.tiles_y * a.tiles_x;
  if (mt <= 0 || mt > 0x7fffffff) return SST_ERR_ARG;
  dim3 grid((unsigned)mt, d->N / BN);
  auto kern = k_l8_tile<BN, EPI>;
  SST_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  kern<<<grid, 128, Cfg::SMEM, st>>>(tmA, tmB, a);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

static bool is_taps233(const SstConvDesc* d) {
  if (d->n_taps != 18) return false;
  for (int i = 0; i < 18; ++i) {
    const int kt = i / 9, ky = (i / 3) % 3, kx = i % 3;
    if (d->taps[i][0] != kt - 1 || d->taps[i][1] != ky - 1 || d->taps[i][2] != kx - 1) return false;
  }
  return true;
}

static int sm_count(int* n) {
  int dev = 0;
  SST_CUDA_TRY(cudaGetDevice(&dev));
  SST_CUDA_TRY(cudaDeviceGetAttribute(n, cudaDevAttrMultiProcessorCount, dev));
  return SST_OK;
}

// kind: 0 = (2,3,3) halo conv, 1 = 1x1 STORE GEMM (TMA-store epilogue), 2 = pixels
static int launch_pair(const SstConvDesc* d, cudaStream_t st, int kind) {
  const bool halo = kind == 0, pix = kind == 2;
  const int nu = pix ? 192 : 256;
  if (d->N % nu != 0 || d->in_W != d->Wt || d->in_H != d->Ht) return SST_ERR_ARG;
  if (halo && (d->t_lo != 0 || d->t_cnt != d->in_T || d->in_T != d->out_T)) return SST_ERR_ARG;
  if (!halo && (d->n_taps != 1 || d->taps[0][1] != 0 || d->taps[0][2] != 0)) return SST_ERR_ARG;
  CUtensorMap tmA, tmB, tmC;
  memset(&tmA, 0, sizeof(tmA));
  memset(&tmB, 0, sizeof(tmB));
  memset(&tmC, 0, sizeof(tmC));
  const uint64_t adims[5] = {(uint64_t)d->in_C, (uint64_t)d->in_W, (uint64_t)d->in_H,
                             (uint64_t)d->in_T, (uint64_t)d->G};
  if (!make_tmap_u8_5d(&tmA, d->in, adims, halo ? pc::PITCH : 8, halo ? pc::HROWS : 16))
    return SST_ERR_ARG;
  if (!make_tmap_u8_2d(&tmB, d->weight, (uint64_t)d->K, (uint64_t)d->N, nu / 2)) return SST_ERR_ARG;
  if (kind == 1) {
    const uint64_t cdims[5] = {(uint64_t)d->N, (uint64_t)d->Wt, (uint64_t)d->Ht,
                               (uint64_t)d->out_T, (uint64_t)d->G};
    if (!make_tmap_u8_5d(&tmC, d->out, cdims, 8, 16)) return SST_ERR_ARG;
  }
  Args a;
  fill_args(a, d, pc::TILE, pc::TILE);
  const int n_blocks = d->N / nu;
  const int64_t units = (int64_t)d->G * d->t_cnt * a.tiles_y * a.tiles_x * n_blocks;
  if (units <= 0 || units > 0x7fffffff) return SST_ERR_ARG;
  int n_sm = 0;
  if (sm_count(&n_sm) != SST_OK) return SST_ERR_CUDA;
  const int64_t pairs = units < n_sm / 2 ? units : n_sm / 2;
  auto kern = halo ? k_l8_pair<true, false> : (pix ? k_l8_pair<false, false, true> : k_l8_pair<false, true>);
  const int smem = halo ? pair_smem<true, false>()
                        : (pix ? pair_smem<false, false, true>() : pair_smem<false, true>());
  SST_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int threads = pix ? pc::pair_threads<true>() : pc::pair_threads<false>();
  kern<<<(unsigned)(2 * pairs), threads, smem, st>>>(tmA, tmB, tmC, a, (int)units, n_blocks);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

}  // namespace l8
}  // namespace sst

#include <cstdlib>

using namespace sst;

extern "C" int sst_lt8_conv(const SstConvDesc* d, void* stream) {
  if (!d || !d->in || !d->weight || !d->bias_i32) return SST_ERR_ARG;
  if (reinterpret_cast<uintptr_t>(d->bias_i32) & 15u) return SST_ERR_ARG;   // int4 bias loads
  if (d->in_C <= 0 || d->in_C % l8::KB != 0) return SST_ERR_ARG;
  if (d->n_taps < 1 || d->n_taps > 27 || d->K != d->n_taps * d->in_C) return SST_ERR_ARG;
  if (d->G <= 0 || d->Ht <= 0 || d->Wt <= 0 || d->t_cnt <= 0) return SST_ERR_ARG;
  if (d->shift < 1 || d->shift > 30) return SST_ERR_ARG;
  for (int i = 0; i < d->n_taps; ++i)
    for (int j = 0; j < 3; ++j)
      if (d->taps[i][j] < -8 || d->taps[i][j] > 8) return SST_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // SST_LT8_GEMM=tile: every layer through the generic tile kernel (A/B, tests)
  const char* mode = getenv("SST_LT8_GEMM");
  const bool tile_only = mode && mode[0] == 't';
  const bool one_by_one = d->n_taps == 1 && d->taps[0][1] == 0 && d->taps[0][2] == 0 &&
                          d->in_W == d->Wt && d->in_H == d->Ht;
  switch (d->epi) {
    case SST_LT_EPI_STORE:
      if (!d->out || d->act < 0 || d->act > 1 || (d->act && !d->act_lut)) return SST_ERR_ARG;
      if ((reinterpret_cast<uintptr_t>(d->out) & 15u) ||
          (d->residual && (reinterpret_cast<uintptr_t>(d->residual) & 15u)) || d->N % 32)
        return SST_ERR_ARG;
      if (!tile_only && d->N % 256 == 0) {
        if (l8::is_taps233(d)) return l8::launch_pair(d, st, 0);
        if (one_by_one) return l8::launch_pair(d, st, 1);
      }
      if (d->N % 128 == 0) return l8::launch_tile<128, SST_LT_EPI_STORE>(d, st);
      return l8::launch_tile<32, SST_LT_EPI_STORE>(d, st);
    case SST_LT_EPI_FSQ:
      if (!d->codes || !d->idx || !d->mask || d->N != 16 || d->t_lo != 0 || d->t_cnt != 2)
        return SST_ERR_ARG;
      return l8::launch_tile<16, SST_LT_EPI_FSQ>(d, st);
    case SST_LT_EPI_PIXELS:
    case SST_LT_EPI_PIXELS_U8:
      if (!d->frames || d->h <= 0 || d->w <= 0 || d->frame_base < 0 ||
          d->frame_base + d->N / 192 > 9 || d->h > d->Ht * 8 || d->w > d->Wt * 8 || d->N % 192)
        return SST_ERR_ARG;
      if (!tile_only && one_by_one) return l8::launch_pair(d, st, 2);
      return l8::launch_tile<192, SST_LT_EPI_PIXELS>(d, st);
    default:
      return SST_ERR_ARG;
  }
}

template <bool kHaar>
static int launch_patchify_band(const float* frames, int G, int H, int W, int s, void* pI, void* pP,
                                void* stream);

extern "C" int sst_lt8_patchify(const float* frames, int G, int H, int W, int s, void* pI, void* pP,
                                void* stream) {
  if (!frames || !pI || !pP || G <= 0 || H <= 0 || W <= 0) return SST_ERR_ARG;
  if (s < 1 || s > 3) return SST_ERR_ARG;
  if ((reinterpret_cast<uintptr_t>(pI) & 15u)) return SST_ERR_ARG;
  const int h = ceil_div(H, s), w = ceil_div(W, s);
  const int Ht = ceil_div(h, 8), Wt = ceil_div(w, 8);
  // s = 1: the band kernel (8-row band staged in shared memory, stored as
  // 16-byte vectors; the Haar kernel without the transform): 1.72 vs 2.82 ms
  // per 32 x 1080p GoPs -- the per-pixel kernel's 3-byte stores dominate when
  // nothing is averaged.  s >= 2: the per-pixel kernel (1.06 vs 1.18 ms at
  // s = 3).  SST_LT8_PATCHIFY=band|pixel overrides (A/B).
  const char* mode = getenv("SST_LT8_PATCHIFY");
  const bool band = mode && mode[0] ? mode[0] == 'b' : s == 1;
  if (band) return launch_patchify_band<false>(frames, G, H, W, s, pI, pP, stream);
  const int threads = 256;
  if ((int64_t)G * 9 > 65535 || Ht * 8 > 65535) return SST_ERR_ARG;
  const dim3 blocks(ceil_div(Wt * 8, threads), Ht * 8, G * 9);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto* i = static_cast<int8_t*>(pI);
  auto* p = static_cast<int8_t*>(pP);
  switch (s) {
    case 1: l8::k_l8_patchify<1><<<blocks, threads, 0, st>>>(frames, G, H, W, h, w, Ht, Wt, i, p); break;
    case 2: l8::k_l8_patchify<2><<<blocks, threads, 0, st>>>(frames, G, H, W, h, w, Ht, Wt, i, p); break;
    default: l8::k_l8_patchify<3><<<blocks, threads, 0, st>>>(frames, G, H, W, h, w, Ht, Wt, i, p); break;
  }
  SST_LAUNCH_CHECK();
  return SST_OK;
}

template <bool kHaar>
static int launch_patchify_band(const float* frames, int G, int H, int W, int s, void* pI, void* pP,
                                void* stream) {
  if (!frames || !pI || !pP || G <= 0 || H <= 0 || W <= 0) return SST_ERR_ARG;
  if (s < 1 || s > 3) return SST_ERR_ARG;
  if ((reinterpret_cast<uintptr_t>(pI) & 15u) || (reinterpret_cast<uintptr_t>(pP) & 15u))
    return SST_ERR_ARG;
  const int h = ceil_div(H, s), w = ceil_div(W, s);
  const int Ht = ceil_div(h, 8), Wt = ceil_div(w, 8);
  if (G > 65535 || Ht > 65535) return SST_ERR_ARG;
  const dim3 blocks(ceil_div(Wt, l8::kHaarTok), Ht, G);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto* i = static_cast<int8_t*>(pI);
  auto* p = static_cast<int8_t*>(pP);
  constexpr int T = l8::kHaarThreads;
  switch (s) {
    case 1: l8::k_l8_patchify_band<1, kHaar><<<blocks, T, 0, st>>>(frames, H, W, h, w, Ht, Wt, i, p); break;
    case 2: l8::k_l8_patchify_band<2, kHaar><<<blocks, T, 0, st>>>(frames, H, W, h, w, Ht, Wt, i, p); break;
    default: l8::k_l8_patchify_band<3, kHaar><<<blocks, T, 0, st>>>(frames, H, W, h, w, Ht, Wt, i, p); break;
  }
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_lt8_patchify_haar(const float* frames, int G, int H, int W, int s, void* pI,
                                     void* pP, void* stream) {
  return launch_patchify_band<true>(frames, G, H, W, s, pI, pP, stream);
}

extern "C" int sst_lt8_attn(const void* qkv, int G, int Ht, int Wt, int D, int shift,
                            const uint8_t* exp_lut, void* out, void* stream) {
  if (!qkv || !out || !exp_lut || G <= 0 || Ht <= 0 || Wt <= 0 || D <= 0 || D % l8::AT_HD)
    return SST_ERR_ARG;
  if (shift < 0 || shift > 30 || G > 65535 || D / l8::AT_HD > 65535) return SST_ERR_ARG;
  if ((reinterpret_cast<uintptr_t>(qkv) & 15u) || (reinterpret_cast<uintptr_t>(out) & 15u))
    return SST_ERR_ARG;
  const int64_t wins = (int64_t)ceil_div(Ht, l8::AT_WIN) * ceil_div(Wt, l8::AT_WIN);
  if (wins > 0x7fffffff) return SST_ERR_ARG;
  dim3 grid((unsigned)wins, D / l8::AT_HD, G);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SST_CUDA_TRY(cudaFuncSetAttribute(l8::k_l8_attn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    l8::AT_SMEM));
  l8::k_l8_attn<<<grid, 128, l8::AT_SMEM, st>>>(static_cast<const int8_t*>(qkv), G, Ht, Wt, D,
                                                shift, exp_lut, static_cast<int8_t*>(out));
  SST_LAUNCH_CHECK();
  return SST_OK;
}

extern "C" int sst_lt8_attn_global(const void* qkv, int G, int Ht, int Wt, int D, int shift,
                                   const uint8_t* exp_lut, void* out, void* stream) {
  if (!qkv || !out || !exp_lut || G <= 0 || Ht <= 0 || Wt <= 0 || D <= 0 || D % l8::AT_HD)
    return SST_ERR_ARG;
  if (shift < 0 || shift > 30 || 2 * (int64_t)G > 65535 || D / l8::AT_HD > 65535) return SST_ERR_ARG;
  if ((reinterpret_cast<uintptr_t>(qkv) & 15u) || (reinterpret_cast<uintptr_t>(out) & 15u))
    return SST_ERR_ARG;
  const int64_t n = (int64_t)Ht * Wt;
  if (n > (1 << 24)) return SST_ERR_ARG;
  dim3 grid((unsigned)((n + 127) / 128), D / l8::AT_HD, 2 * G);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const char* mode = getenv("SST_AG");
  CUtensorMap tq;
  memset(&tq, 0, sizeof(tq));
  if (!(mode && mode[0] == 'o') && 2 * (int64_t)G * n < (1ll << 31) &&
      make_tmap_u8_2d(&tq, qkv, (uint64_t)3 * D, (uint64_t)2 * G * n, 128)) {
    static bool attr = false;
    if (!attr) {
      SST_CUDA_TRY(cudaFuncSetAttribute(l8::k_l8_attn_global_tma,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, l8::AG2_SMEM));
      attr = true;
    }
    l8::k_l8_attn_global_tma<<<grid, 128, l8::AG2_SMEM, st>>>(tq, G, (int)n, D, shift, exp_lut,
                                                              static_cast<int8_t*>(out));
    SST_LAUNCH_CHECK();
    return SST_OK;
  }
  SST_CUDA_TRY(cudaFuncSetAttribute(l8::k_l8_attn_global, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    l8::AG_SMEM));
  l8::k_l8_attn_global<<<grid, 128, l8::AG_SMEM, st>>>(static_cast<const int8_t*>(qkv), G, (int)n,
                                                       D, shift, exp_lut, static_cast<int8_t*>(out));
  SST_LAUNCH_CHECK();
  return SST_OK;
}
