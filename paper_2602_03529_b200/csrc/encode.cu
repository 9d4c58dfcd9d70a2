// K1: scale_gop(down) + encode_gop + token_similarity, fused.
//
// Reference: codec.py:202-214 (downscale_frame), codec.py:99-128
// (_pad_to_block/_blockify/_tokenize_image), codec.py:143-157 (encode_gop),
// selection.py:33-52 (token_similarity).
//
// One CTA owns one token row x TPB token columns of one GoP.  It streams the
// 9 full-resolution frame tiles it needs (8s rows x TPB*8s pixels x RGB)
// through a 4-deep TMA ring (mbarrier completion), box-filters them in
// float64 into registers (frame 0 -> I source, frames 1..8 -> running P sum),
// then runs the ducc0-exact 8x8 DCT on the two working-resolution blocks per
// token and channel, and finally the cosine similarity of each token pair.
// HBM traffic is one read of every input pixel plus the token write.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "dct8.cuh"
#include "tma.cuh"

namespace sst {

template <int S>
struct EncCfg {
  static constexpr int TPB = (S == 3) ? 3 : 4;      // tokens per CTA
  static constexpr int R = 8 * S;                   // full-res rows per tile
  static constexpr int IN = TPB * 8 * S * 3;        // floats per tile row
  static constexpr int NT = 64 * TPB;               // one thread per working pixel
  // TMA ring depth: s=3 tiles are 20 KB, and a 4-deep ring (83 KB) capped
  // residency at 2 CTAs / SM; 3 deep (62 KB, 3 CTAs) runs K1 at 7.2 instead
  // of 6.75 TB/s (scripts/k1_micro.py: 0.99 vs 1.06 ms per 32 GoPs)
  static constexpr int NST = (S == 3) ? 3 : 4;
  static constexpr int TILE = R * IN;               // floats per tile
  static constexpr int RING_BYTES = NST * TILE * 4;
  static constexpr int IMG_D = 2 * 8 * 8 * TPB * 3;            // imgbuf doubles
  static constexpr int S1_D = 2 * TPB * 3 * 3 * 8;             // stage-1 doubles
  static constexpr int TOK_D = 2 * TPB * kChannels;            // token doubles
  static constexpr int DCT_BYTES = (IMG_D + S1_D + TOK_D) * 8;
  static constexpr int MAIN_BYTES = RING_BYTES > DCT_BYTES ? RING_BYTES : DCT_BYTES;
  static constexpr int SMEM = MAIN_BYTES + 128 + NST * 8;
};

struct EncArgs {
  const float* frames;
  int G, H, W, h, w, Ht, Wt;
  double* tok;
  double* sim;
  float* work;   // optional: the working frames [G][9][h][w][3] (scale_gop(down))
};

// numpy pairwise order for a 12-long reduction (8-way unrolled block + tail)
__device__ __forceinline__ double pairwise12(const double* x) {
  double r = ((x[0] + x[1]) + (x[2] + x[3])) + ((x[4] + x[5]) + (x[6] + x[7]));
  r = r + x[8];
  r = r + x[9];
  r = r + x[10];
  r = r + x[11];
  return 0.0 + r;  // add.reduce identity start
}

__device__ __forceinline__ double cosine12(const double* p, const double* i) {
  double a[12], b[12], c[12];
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    a[k] = p[k] * i[k];
    b[k] = p[k] * p[k];
    c[k] = i[k] * i[k];
  }
  double dot = pairwise12(a);
  double pn = sqrt(pairwise12(b));
  double in = sqrt(pairwise12(c));
  double denom = pn * in;
  double s = denom > 0.0 ? dot / denom : 0.0;
  if (pn == 0.0 && in == 0.0) s = 1.0;
  return clip_pm1(s);
}

template <int S, bool kTMA>
__global__ void __launch_bounds__(EncCfg<S>::NT)
    k_encode(const __grid_constant__ CUtensorMap tmap, EncArgs a) {
  using C = EncCfg<S>;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  float* ring = reinterpret_cast<float*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + C::MAIN_BYTES);  // mbarriers

  const int tid = threadIdx.x;
  const int tx0 = blockIdx.x * C::TPB;
  const int ty = blockIdx.y;
  const int g = blockIdx.z;
  const int row0 = ty * C::R;                 // first full-res row of the tile
  const int col0 = tx0 * 8 * S;               // first full-res pixel column
  const size_t frame_elems = (size_t)a.H * a.W * 3;
  const float* gop = a.frames + (size_t)g * kGop * frame_elems;

  if (kTMA && tid == 0) {
    for (int st = 0; st < C::NST; ++st) mbar_init(&full[st], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (kTMA && tid == 0) {
    for (int f = 0; f < C::NST; ++f) {
      mbar_expect_tx(&full[f], C::TILE * 4);
      tma_load_3d(ring + f * C::TILE, &tmap, col0 * 3, row0, g * kGop + f, &full[f]);
    }
  }

  // this thread's working pixel (clamped = working-res edge replication,
  // codec.py:99-105) and its s x s full-res window (clamped = full-res edge
  // replication, codec.py:209-211), as offsets inside a tile
  const int wy = tid / (8 * C::TPB);
  const int wx = tid % (8 * C::TPB);
  const int ay = min(ty * 8 + wy, a.h - 1);
  const int ax = min(tx0 * 8 + wx, a.w - 1);
  int off[S * S];
#pragma unroll
  for (int j = 0; j < S; ++j) {
    int r = min(ay * S + j, a.H - 1) - row0;
#pragma unroll
    for (int l = 0; l < S; ++l) {
      int c = min(ax * S + l, a.W - 1) - col0;
      off[j * S + l] = r * C::IN + c * 3;
    }
  }

  float ival[3];
  double pacc[3];
  constexpr double div_ss = (double)(S * S);
  // the working pixel this thread box-filters, written out when asked for
  // (the residual layer's `working` GoP, session.py:173-189) -- only real
  // pixels, not the block padding's edge replicas
  const size_t work_frame = (size_t)a.h * a.w * 3;
  float* wout = nullptr;
  if (a.work != nullptr && ty * 8 + wy < a.h && tx0 * 8 + wx < a.w)
    wout = a.work + (size_t)g * kGop * work_frame + ((size_t)(ty * 8 + wy) * a.w + tx0 * 8 + wx) * 3;

  for (int f = 0; f < kGop; ++f) {
    const int st = f % C::NST;
    float* tile = ring + st * C::TILE;
    if (kTMA) {
      mbar_wait(&full[st], (f / C::NST) & 1);
    } else {
      // plain cooperative load of the in-bounds part of the tile
      const float* src = gop + (size_t)f * frame_elems;
      for (int e = tid; e < C::TILE; e += C::NT) {
        int r = e / C::IN, c = e % C::IN;
        int gr = row0 + r, gc = col0 * 3 + c;
        if (gr < a.H && gc < a.W * 3) tile[e] = __ldg(src + (size_t)gr * a.W * 3 + gc);
      }
      __syncthreads();
    }
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      // numpy add.reduce starts from the identity 0.0 (matters only for -0.0)
      double acc = 0.0 + (double)tile[off[0] + ch];
#pragma unroll
      for (int q = 1; q < S * S; ++q) acc = acc + (double)tile[off[q] + ch];
      float wv = __double2float_rn(acc / div_ss);     // Frame float32 storage
      if (wout != nullptr) wout[(size_t)f * work_frame + ch] = wv;
      if (f == 0) {
        ival[ch] = wv;
      } else if (f == 1) {
        pacc[ch] = 0.0 + (double)wv;
      } else {
        pacc[ch] = pacc[ch] + (double)wv;              // codec.py:151-152, sequential
      }
    }
    __syncthreads();  // everyone is done with this stage
    if (kTMA && tid == 0 && f + C::NST < kGop) {
      mbar_expect_tx(&full[st], C::TILE * 4);
      tma_load_3d(tile, &tmap, col0 * 3, row0, g * kGop + f + C::NST, &full[st]);
    }
  }

  // ---- 8x8 DCT of the I and P working blocks (ring is free now) ----
  double* img = reinterpret_cast<double*>(smem_raw);                 // [2][8][8*TPB][3]
  double* s1 = img + C::IMG_D;                                       // [2][TPB][3][3][8]
  double* tk = s1 + C::S1_D;                                         // [2][TPB][12]
  {
    const int base = (wy * 8 * C::TPB + wx) * 3;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      img[base + ch] = (double)ival[ch];
      img[8 * 8 * C::TPB * 3 + base + ch] = pacc[ch] / 8.0;
    }
  }
  __syncthreads();
  // stage 1: along y (axis -2) for every block column, fct = 1/16
  for (int it = tid; it < 48 * C::TPB; it += C::NT) {
    int im = it / (24 * C::TPB);
    int rem = it % (24 * C::TPB);
    int t = rem / 24, ch = (rem % 24) / 8, x = rem % 8;
    double c[8];
    const double* src = img + im * (8 * 8 * C::TPB * 3) + (t * 8 + x) * 3 + ch;
#pragma unroll
    for (int y = 0; y < 8; ++y) c[y] = src[y * 8 * C::TPB * 3];
    dct2_8<true>(c, 1.0 / 16.0);
    double* dst = s1 + ((im * C::TPB + t) * 3 + ch) * 24;
    dst[x] = c[0];
    dst[8 + x] = c[1];
    dst[16 + x] = c[2];
  }
  __syncthreads();
  // stage 2: along x for rows y = 0, 1, 2; keep (0,0) (0,1) (1,0) (2,0)
  for (int it = tid; it < 18 * C::TPB; it += C::NT) {
    int im = it / (9 * C::TPB);
    int rem = it % (9 * C::TPB);
    int t = rem / 9, ch = (rem % 9) / 3, yk = rem % 3;
    double c[8];
    const double* src = s1 + ((im * C::TPB + t) * 3 + ch) * 24 + yk * 8;
#pragma unroll
    for (int x = 0; x < 8; ++x) c[x] = src[x];
    dct2_8<false>(c, 1.0);
    double* dst = tk + (im * C::TPB + t) * kChannels + ch * 4;
    if (yk == 0) {
      dst[0] = c[0];
      dst[1] = c[1];
    } else {
      dst[yk + 1] = c[0];
    }
  }
  __syncthreads();
  for (int e = tid; e < 2 * C::TPB * kChannels; e += C::NT) {
    int im = e / (C::TPB * kChannels);
    int t = (e / kChannels) % C::TPB;
    int k = e % kChannels;
    int tx = tx0 + t;
    if (tx < a.Wt)
      a.tok[((((size_t)g * 2 + im) * a.Ht + ty) * a.Wt + tx) * kChannels + k] = tk[e];
  }
  if (a.sim != nullptr && tid < C::TPB && tx0 + tid < a.Wt) {
    const double* iv = tk + tid * kChannels;
    const double* pv = tk + (C::TPB + tid) * kChannels;
    a.sim[((size_t)g * a.Ht + ty) * a.Wt + tx0 + tid] = cosine12(pv, iv);
  }
}

// ---- K1 over raw-rgb24 frames (load_raw_video fused) ----
//
// The reference CLI ingests raw-rgb24 files: every byte q becomes the float32
// sample f(q) = float32(q) / 255 (video.py:130-135; a float32 array divided by
// a Python float stays float32, correctly rounded).  K1u8 reads the bytes --
// a quarter of the float32 frames' HBM traffic -- and box-filters f(q)
// exactly.  q / 255 in binary is q's 8 bits repeated forever, so
// floor(q/255 * 2^32) = q * 0x01010101, and rounding to float32's 24
// significant bits always rounds UP (the first dropped bit is q's leading
// one, the rest of the expansion is non-zero), giving the identity
//     f(q) * 2^32 = q * 0x01010100 + g(q),   g(q) = 2^(msb(q) + 1), g(0) = 0
// (checked for all 256 values).  So the window sum is
//     sum f = (0x01010100 * sum q + sum g) * 2^-32,
// exact in float64 -- the value numpy's float64 sum reaches in any order,
// since every partial sum of <= 9 such samples is exact.  One 32-bit table
// entry T(q) = q << 16 | g(q) per byte gives both sums with one 32-bit add
// (sum q, sum g < 2^16 for <= 9 terms).  T lives in shared memory replicated
// 32x (entry q of copy c at word 32q + c, lane l reads copy l): the lookups
// are bank-conflict free.
//
// Work mapping: each thread box-filters a QUAD of 4 horizontally adjacent
// working pixels of one working row, so the quad's s rows x 12s bytes are
// word-aligned in the tile and read as 3s 32-bit words.  A CTA covers one
// token row x 8 token columns (128 threads); the 9 frame tiles stream
// through a cp.async ring (16-byte copies) with a padded row pitch.
constexpr int kU8Tpb = 8;

template <int S>
struct EncU8Cfg {
  static constexpr int TPB = kU8Tpb;                // tokens per CTA
  static constexpr int R = 8 * S;                   // full-res rows per tile
  static constexpr int IN = TPB * 8 * S * 3;        // bytes per tile row
  static constexpr int INP = IN + 16;               // padded pitch
  static constexpr int NQ = TPB * 8 / 4;            // quads per working row
  static constexpr int NT = 8 * NQ;                 // threads (128)
  static constexpr int QB = 12 * S;                 // bytes per quad row segment
  static constexpr int NST = 3;                     // ring depth
  static constexpr int TILE = R * INP;              // bytes per ring stage
  static constexpr int RING = NST * TILE;
  static constexpr int IMG_D = 2 * 8 * 8 * TPB * 3;
  static constexpr int S1_D = 2 * TPB * 3 * 3 * 8;
  static constexpr int TOK_D = 2 * TPB * kChannels;
  static constexpr int DCT_BYTES = (IMG_D + S1_D + TOK_D) * 8;
  static constexpr int LUT_WORDS = 256 * 32;
  // the table follows the ring; the DCT stage (after the frame loop) reuses
  // both, so the footprint is max(ring + table, DCT) -- 52 KB at s = 1, 2:
  // 4 CTAs per SM (s = 3: 75 KB, 3 CTAs)
  static constexpr int LUT_OFF = (RING + 127) / 128 * 128;
  static constexpr int SMEM = LUT_OFF + LUT_WORDS * 4 > DCT_BYTES ? LUT_OFF + LUT_WORDS * 4 : DCT_BYTES;
  static constexpr int MIN_CTAS = S == 3 ? 3 : 4;
};

struct EncU8Args {
  const uint8_t* frames;
  int G, H, W, h, w, Ht, Wt;
  double* tok;
  double* sim;
  float* work;
  int aligned;   // frames and rows 16-byte aligned: cp.async 16-byte tile copies
};

template <int S, bool kWork>
__global__ void __launch_bounds__(EncU8Cfg<S>::NT, EncU8Cfg<S>::MIN_CTAS) k_encode_u8(EncU8Args a) {
  using C = EncU8Cfg<S>;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* ring = smem_raw;
  uint32_t* lut = reinterpret_cast<uint32_t*>(smem_raw + C::LUT_OFF);
  const int tid = threadIdx.x, lane = tid & 31;
  const int tx0 = blockIdx.x * C::TPB;
  const int ty = blockIdx.y;
  const int g = blockIdx.z;
  const int row0 = ty * C::R;
  const int col0 = tx0 * 8 * S;
  const size_t frame_bytes = (size_t)a.H * a.W * 3;
  const uint8_t* gop = a.frames + (size_t)g * kGop * frame_bytes;

  // this thread's 16-byte chunks of a tile (the same for every frame):
  // smem offset and frame-relative global offset, -1 when outside the frame
  constexpr int kChunks = C::IN / 16;
  constexpr int kCpt = (C::R * kChunks + C::NT - 1) / C::NT;
  int c_smem[kCpt], c_glob[kCpt];
#pragma unroll
  for (int k = 0; k < kCpt; ++k) {
    const int e = tid + k * C::NT;
    const int r = e / kChunks, c = e % kChunks;
    const int gr = row0 + r, gb = col0 * 3 + c * 16;
    const bool ok = e < C::R * kChunks && gr < a.H && gb < a.W * 3;   // W*3 % 16 == 0: chunks whole
    c_smem[k] = ok ? r * C::INP + c * 16 : -1;
    c_glob[k] = gr * a.W * 3 + gb;
  }
  const uint32_t ring_u32 = smem_u32(ring);
  // tile f -> ring stage f % NST: rows row0..row0+R-1 (< H), bytes col0*3..
  auto load_tile = [&](int f) {
    uint8_t* dst = ring + (f % C::NST) * C::TILE;
    const uint8_t* src = gop + (size_t)f * frame_bytes;
    if (a.aligned) {
      const uint32_t d0 = ring_u32 + (f % C::NST) * C::TILE;
#pragma unroll
      for (int k = 0; k < kCpt; ++k)
        if (c_smem[k] >= 0)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d0 + c_smem[k]), "l"(src + c_glob[k])
                       : "memory");
    } else {
      for (int e = tid; e < C::R * C::IN; e += C::NT) {
        const int r = e / C::IN, c = e % C::IN;
        const int gr = row0 + r, gb = col0 * 3 + c;
        if (gr < a.H && gb < a.W * 3) dst[r * C::INP + c] = __ldg(src + (size_t)gr * a.W * 3 + gb);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll 1
  for (int f = 0; f < C::NST; ++f) load_tile(f);

  // T(q) table: entry q's 32 copies are 128 contiguous bytes, written as
  // 8 x 16-byte stores (consecutive threads: consecutive 16-byte chunks)
  for (int e = tid; e < 256 * 8; e += C::NT) {
    const uint32_t q = (uint32_t)e >> 3;
    const uint32_t t = (q << 16) | (q ? 2u << (31 - __clz(q)) : 0u);
    reinterpret_cast<uint4*>(lut)[e] = make_uint4(t, t, t, t);
  }

  const int wy = tid / C::NQ, qi = tid % C::NQ;
  const int ay = min(ty * 8 + wy, a.h - 1);
  const int px0 = tx0 * 8 + qi * 4;                // first working pixel of the quad
  const bool interior = px0 + 3 < a.w && (px0 + 4) * S <= a.W;
  const uint32_t lut_lane = smem_u32(lut) + 4u * lane;    // this lane's copy
  constexpr double div_ss = (double)(S * S);
  const size_t work_frame = (size_t)a.h * a.w * 3;
  const bool wrow = kWork && ty * 8 + wy < a.h;
  double ival[4][3];                               // float32 values, held as float64
  double pacc[4][3];

#pragma unroll 1
  for (int f = 0; f < kGop; ++f) {
    asm volatile("cp.async.wait_group %0;" ::"n"(C::NST - 1) : "memory");
    __syncthreads();                               // tile f (and, at f = 0, the table) visible
    const uint8_t* tile = ring + (f % C::NST) * C::TILE;
    uint32_t acc[4][3];                            // sum q << 16 | sum g per (pixel, channel)
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) acc[p][ch] = 0;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const int r = min(ay * S + j, a.H - 1) - row0;
      if (interior) {
        const uint32_t* wp = reinterpret_cast<const uint32_t*>(tile + r * C::INP + qi * C::QB);
        uint32_t wd[3 * S];
#pragma unroll
        for (int k = 0; k < 3 * S; ++k) wd[k] = wp[k];
#pragma unroll
        for (int b = 0; b < 12 * S; ++b) {         // byte b: pixel b / 3S, column (b % 3S) / 3, channel b % 3
          // (an ALU form without the table -- float(q) as (2^23 + q) - 2^23,
          // g(q) from its exponent -- measured slower at every mix)
          const uint32_t q = __byte_perm(wd[b >> 2], 0u, 0x4440u + (b & 3));
          uint32_t t;
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(t) : "r"(lut_lane + q * 128u));
          acc[b / (3 * S)][b % 3] += t;
        }
      } else {
        const uint8_t* rp = tile + r * C::INP;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const int ax = min(px0 + p, a.w - 1);
#pragma unroll
          for (int l = 0; l < S; ++l) {
            const int c = min(ax * S + l, a.W - 1) - col0;
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) acc[p][ch] += lut[((uint32_t)rp[c * 3 + ch] << 5) + lane];
          }
        }
      }
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      float* wout = nullptr;
      if (kWork && wrow && px0 + p < a.w)
        wout = a.work + (size_t)g * kGop * work_frame + (size_t)f * work_frame +
               ((size_t)(ty * 8 + wy) * a.w + px0 + p) * 3;
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        // N = 2^32 * sum f(q) = 0x01010100 * sum q + sum g  (< 2^36), as a
        // float64 without the XU: 2^52 + N has N as its low mantissa bits
        const uint64_t n = (uint64_t)(acc[p][ch] >> 16) * 0x01010100u + (acc[p][ch] & 0xFFFFu);
        const double dn = __dadd_rn(__hiloint2double((int)((uint32_t)(n >> 32) | 0x43300000u), (int)(uint32_t)n),
                                    -4503599627370496.0);
        // float32(float64(sum / s^2)) (codec.py:212-214), sum = N 2^-32.
        // s = 1, 2: the division is exact, so a multiply by 2^-32 / s^2 is
        // too.  s = 3: N / 9 stays >= 2^(e-24) / 9 away from every float32
        // rounding tie (m + 1/2) 2^(e-23) (9 is odd: |N 2^k - 9 m'| >= 1), far
        // beyond float64's error, so rounding any float64 approximation
        // within a few ulps -- the product with float64(2^-32 / 9) -- to
        // float32 gives the float of the correctly rounded quotient.
        const double x = __dmul_rn(dn, 0x1p-32 / div_ss);
        // ... rounded to float32 precision in float64 arithmetic (no XU):
        // (x + c) - c with c = 1.5 * 2^(e(x) + 29) rounds x to a multiple of
        // its float32 ulp 2^(e-23), half to even; x is 0 or in [2^-12, 1],
        // so the result is a normal float32 (also when it rounds up to the
        // next binade)
        const uint32_t xhi = (uint32_t)__double2hiint(x);
        const double c = __hiloint2double((int)((xhi & 0x7FF00000u) + (29u << 20) + 0x00080000u), 0);
        const double xr = __dadd_rn(__dadd_rn(x, c), -c);
        if (kWork && wout != nullptr) wout[ch] = (float)xr;        // exact
        if (f == 0) ival[p][ch] = xr;
        else if (f == 1) pacc[p][ch] = 0.0 + xr;
        else pacc[p][ch] = pacc[p][ch] + xr;                        // codec.py:151-152
      }
    }
    __syncthreads();                               // stage f % NST free
    if (f + C::NST < kGop) load_tile(f + C::NST);
    else asm volatile("cp.async.commit_group;" ::: "memory");   // keep the group count uniform
  }

  // ---- 8x8 DCT of the I and P working blocks (the ring is free) ----
  double* img = reinterpret_cast<double*>(smem_raw);                 // [2][8][8*TPB][3]
  double* s1 = img + C::IMG_D;                                       // [2][TPB][3][3][8]
  double* tk = s1 + C::S1_D;                                         // [2][TPB][12]
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int base = (wy * 8 * C::TPB + qi * 4 + p) * 3;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      img[base + ch] = ival[p][ch];
      img[8 * 8 * C::TPB * 3 + base + ch] = pacc[p][ch] / 8.0;
    }
  }
  __syncthreads();
  for (int it = tid; it < 48 * C::TPB; it += C::NT) {
    int im = it / (24 * C::TPB);
    int rem = it % (24 * C::TPB);
    int t = rem / 24, ch = (rem % 24) / 8, x = rem % 8;
    double c[8];
    const double* src = img + im * (8 * 8 * C::TPB * 3) + (t * 8 + x) * 3 + ch;
#pragma unroll
    for (int y = 0; y < 8; ++y) c[y] = src[y * 8 * C::TPB * 3];
    dct2_8<true>(c, 1.0 / 16.0);
    double* dst = s1 + ((im * C::TPB + t) * 3 + ch) * 24;
    dst[x] = c[0];
    dst[8 + x] = c[1];
    dst[16 + x] = c[2];
  }
  __syncthreads();
  for (int it = tid; it < 18 * C::TPB; it += C::NT) {
    int im = it / (9 * C::TPB);
    int rem = it % (9 * C::TPB);
    int t = rem / 9, ch = (rem % 9) / 3, yk = rem % 3;
    double c[8];
    const double* src = s1 + ((im * C::TPB + t) * 3 + ch) * 24 + yk * 8;
#pragma unroll
    for (int x = 0; x < 8; ++x) c[x] = src[x];
    dct2_8<false>(c, 1.0);
    double* dst = tk + (im * C::TPB + t) * kChannels + ch * 4;
    if (yk == 0) {
      dst[0] = c[0];
      dst[1] = c[1];
    } else {
      dst[yk + 1] = c[0];
    }
  }
  __syncthreads();
  for (int e = tid; e < 2 * C::TPB * kChannels; e += C::NT) {
    int im = e / (C::TPB * kChannels);
    int t = (e / kChannels) % C::TPB;
    int k = e % kChannels;
    int tx = tx0 + t;
    if (tx < a.Wt)
      a.tok[((((size_t)g * 2 + im) * a.Ht + ty) * a.Wt + tx) * kChannels + k] = tk[e];
  }
  if (a.sim != nullptr && tid < C::TPB && tx0 + tid < a.Wt) {
    const double* iv = tk + tid * kChannels;
    const double* pv = tk + (C::TPB + tid) * kChannels;
    a.sim[((size_t)g * a.Ht + ty) * a.Wt + tx0 + tid] = cosine12(pv, iv);
  }
}

template <int S>
static int launch_encode_u8(const uint8_t* frames, int G, int H, int W, double* tok, double* sim,
                            float* work, cudaStream_t stream) {
  using C = EncU8Cfg<S>;
  EncU8Args a;
  a.frames = frames;
  a.G = G; a.H = H; a.W = W;
  a.h = ceil_div(H, S);
  a.w = ceil_div(W, S);
  a.Ht = ceil_div(a.h, kBlock);
  a.Wt = ceil_div(a.w, kBlock);
  a.tok = tok;
  a.sim = sim;
  a.work = work;
  a.aligned = (reinterpret_cast<uintptr_t>(frames) & 15u) == 0 && ((int64_t)W * 3) % 16 == 0;
  if (a.Ht > 65535 || G > 65535) return SST_ERR_ARG;
  dim3 grid(ceil_div(a.Wt, C::TPB), a.Ht, G);
  auto kern = work != nullptr ? k_encode_u8<S, true> : k_encode_u8<S, false>;
  SST_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  kern<<<grid, C::NT, C::SMEM, stream>>>(a);
  SST_LAUNCH_CHECK();
  return SST_OK;
}

// ---- standalone box downscale (downscale_frame, codec.py:202-214) ----
template <int S>
__global__ void k_downscale(const float* __restrict__ src, int64_t n, int H, int W, int h, int w,
                            float* __restrict__ dst) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = n * h * w;
  if (idx >= total) return;
  int x = (int)(idx % w);
  int64_t t = idx / w;
  int y = (int)(t % h);
  int64_t f = t / h;
  const float* fr = src + f * (int64_t)H * W * 3;
  float* out = dst + idx * 3;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      int r = min(y * S + j, H - 1);
#pragma unroll
      for (int l = 0; l < S; ++l) {
        int c = min(x * S + l, W - 1);
        double v = (double)__ldg(fr + ((int64_t)r * W + c) * 3 + ch);
        acc = acc + v;
      }
    }
    out[ch] = __double2float_rn(acc / (double)(S * S));
  }
}

template <int S>
static int launch_encode(const float* frames, int G, int H, int W, double* tok, double* sim, float* work,
                         cudaStream_t stream) {
  using C = EncCfg<S>;
  EncArgs a;
  a.frames = frames;
  a.G = G; a.H = H; a.W = W;
  a.h = ceil_div(H, S);
  a.w = ceil_div(W, S);
  a.Ht = ceil_div(a.h, kBlock);
  a.Wt = ceil_div(a.w, kBlock);
  a.tok = tok;
  a.sim = sim;
  a.work = work;
  if (a.Ht > 65535 || G > 65535) return SST_ERR_ARG;
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  bool use_tma = make_tmap_f32_3d(&tmap, frames, (uint64_t)W * 3, (uint64_t)H, (uint64_t)G * kGop,
                                  C::IN, C::R);
  dim3 grid(ceil_div(a.Wt, C::TPB), a.Ht, G);
  if (use_tma) {
    SST_CUDA_TRY(cudaFuncSetAttribute(k_encode<S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      C::SMEM));
    k_encode<S, true><<<grid, C::NT, C::SMEM, stream>>>(tmap, a);
  } else {
    SST_CUDA_TRY(cudaFuncSetAttribute(k_encode<S, false>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    k_encode<S, false><<<grid, C::NT, C::SMEM, stream>>>(tmap, a);
  }
  SST_LAUNCH_CHECK();
  return SST_OK;
}

}  // namespace sst

using namespace sst;

extern "C" int sst_encode_work(const float* frames, int G, int H, int W, int s, double* tok,
                               double* sim, float* work, void* stream) {
  if (!frames || !tok || G <= 0 || H <= 0 || W <= 0) return SST_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (s) {
    case 1: return launch_encode<1>(frames, G, H, W, tok, sim, work, st);
    case 2: return launch_encode<2>(frames, G, H, W, tok, sim, work, st);
    case 3: return launch_encode<3>(frames, G, H, W, tok, sim, work, st);
    default: return SST_ERR_ARG;
  }
}

extern "C" int sst_encode_u8(const uint8_t* frames, int G, int H, int W, int s, double* tok,
                             double* sim, float* work, void* stream) {
  if (!frames || !tok || G <= 0 || H <= 0 || W <= 0) return SST_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (s) {
    case 1: return launch_encode_u8<1>(frames, G, H, W, tok, sim, work, st);
    case 2: return launch_encode_u8<2>(frames, G, H, W, tok, sim, work, st);
    case 3: return launch_encode_u8<3>(frames, G, H, W, tok, sim, work, st);
    default: return SST_ERR_ARG;
  }
}

extern "C" int sst_encode(const float* frames, int G, int H, int W, int s, double* tok, double* sim,
                          void* stream) {
  return sst_encode_work(frames, G, H, W, s, tok, sim, nullptr, stream);
}

extern "C" int sst_downscale(const float* frames, int64_t n, int H, int W, int s, float* out,
                             void* stream) {
  if (!frames || !out || n <= 0 || H <= 0 || W <= 0) return SST_ERR_ARG;
  if (s != 2 && s != 3) return SST_ERR_ARG;
  int h = ceil_div(H, s), w = ceil_div(W, s);
  int64_t total = n * h * w;
  int threads = 256;
  int64_t blocks = ceil_div64(total, threads);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (s == 2)
    k_downscale<2><<<(unsigned)blocks, threads, 0, st>>>(frames, n, H, W, h, w, out);
  else
    k_downscale<3><<<(unsigned)blocks, threads, 0, st>>>(frames, n, H, W, h, w, out);
  SST_LAUNCH_CHECK();
  return SST_OK;
}
