// 8-point orthonormal DCT-II / DCT-III, bit-identical to the reference's
// scipy.fft.dctn / idctn (codec.py:123, codec.py:138).
//
// scipy 1.18 evaluates these with ducc0's T_dcst23 on an FFTPACK-style real
// FFT (radix-2 pass ido=4 + radix-4 pass ido=1,l1=2).  The operation sequence
// and the twiddle doubles below reproduce it exactly (ducc0's UnityRoots use
// octant symmetry, so e.g. the pi/4 twiddle is sin(fl(pi/4)), one ulp under
// the correctly rounded cos(pi/4)).  Requires -fmad=false (no FMA
// contraction).  The CPU statement of the same algorithm, pinned against
// scipy, lives in oracle/dct8.py.
#pragma once

namespace sst {

struct Dct8 {
  static constexpr double T0 = 0.9807852804032304;
  static constexpr double T1 = 0.9238795325112867;
  static constexpr double T2 = 0.8314696123025452;
  static constexpr double T3 = 0.7071067811865475;
  static constexpr double T4 = 0.5555702330196022;
  static constexpr double T5 = 0.3826834323650898;
  static constexpr double T6 = 0.19509032201612825;
  static constexpr double W8R = 0.7071067811865475;
  static constexpr double W8I = 0.7071067811865476;
  static constexpr double SQRT2 = 1.4142135623730951;
  static constexpr double HALF_SQRT2 = 0.7071067811865476;  // SQRT2 * 0.5
  static constexpr double TWO_T3 = 1.414213562373095;       // 2 * T3
};

// Backward real FFT, half-complex in -> real out (in place, 8 values).
__device__ __forceinline__ void rfft8_backward(double* c) {
  double d0 = c[0] + c[7];
  double d4 = c[0] - c[7];
  double d3 = 2.0 * c[3];
  double d7 = -2.0 * c[4];
  double d1 = c[1] + c[5];
  double tr2 = c[1] - c[5];
  double ti2 = c[2] + c[6];
  double d2 = c[2] - c[6];
  double d6 = Dct8::W8R * ti2 + Dct8::W8I * tr2;
  double d5 = Dct8::W8R * tr2 - Dct8::W8I * ti2;
  // radix-4 pass, k = 0 uses d0..d3, k = 1 uses d4..d7
  {
    double s = d0 + d3, m = d0 - d3, t1 = 2.0 * d1, t2 = 2.0 * d2;
    c[0] = s + t1; c[4] = s - t1; c[6] = m + t2; c[2] = m - t2;
  }
  {
    double s = d4 + d7, m = d4 - d7, t1 = 2.0 * d5, t2 = 2.0 * d6;
    c[1] = s + t1; c[5] = s - t1; c[7] = m + t2; c[3] = m - t2;
  }
}

// Forward real FFT, real in -> half-complex out (in place, 8 values).
__device__ __forceinline__ void rfft8_forward(double* c) {
  double d[8];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    double s31 = c[k + 6] + c[k + 2];
    d[4 * k + 2] = c[k + 6] - c[k + 2];
    double s02 = c[k] + c[k + 4];
    d[4 * k + 1] = c[k] - c[k + 4];
    d[4 * k] = s02 + s31;
    d[4 * k + 3] = s02 - s31;
  }
  double tr2 = Dct8::W8R * d[5] + Dct8::W8I * d[6];
  double ti2 = Dct8::W8R * d[6] - Dct8::W8I * d[5];
  c[0] = d[0] + d[4];
  c[7] = d[0] - d[4];
  c[4] = -d[7];
  c[3] = d[3];
  c[1] = d[1] + tr2;
  c[5] = d[1] - tr2;
  c[2] = ti2 + d[2];
  c[6] = ti2 - d[2];
}

// DCT-II ortho along 8 values; fct is the ducc0 normalisation (1/16 for the
// first axis of dctn, 1 for the second).  In place.
template <bool kScale>
__device__ __forceinline__ void dct2_8(double* c, double fct) {
  c[0] = c[0] * 2.0;
  c[7] = c[7] * 2.0;
#pragma unroll
  for (int k = 1; k < 7; k += 2) {
    double hi = c[k + 1];
    c[k + 1] = hi - c[k];
    c[k] = c[k] + hi;
  }
  rfft8_backward(c);
  if (kScale) {
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = c[k] * fct;
  }
  {
    double t1 = Dct8::T0 * c[7] + Dct8::T6 * c[1];
    double t2 = Dct8::T0 * c[1] - Dct8::T6 * c[7];
    c[1] = 0.5 * (t1 + t2); c[7] = 0.5 * (t1 - t2);
  }
  {
    double t1 = Dct8::T1 * c[6] + Dct8::T5 * c[2];
    double t2 = Dct8::T1 * c[2] - Dct8::T5 * c[6];
    c[2] = 0.5 * (t1 + t2); c[6] = 0.5 * (t1 - t2);
  }
  {
    double t1 = Dct8::T2 * c[5] + Dct8::T4 * c[3];
    double t2 = Dct8::T2 * c[3] - Dct8::T4 * c[5];
    c[3] = 0.5 * (t1 + t2); c[5] = 0.5 * (t1 - t2);
  }
  c[4] = c[4] * Dct8::T3;
  c[0] = c[0] * Dct8::HALF_SQRT2;
}

// DCT-III ortho (inverse of dct2_8) along 8 values, in place.
template <bool kScale>
__device__ __forceinline__ void dct3_8(double* c, double fct) {
  c[0] = c[0] * Dct8::SQRT2;
  {
    double t1 = c[1] + c[7], t2 = c[1] - c[7];
    c[1] = Dct8::T0 * t2 + Dct8::T6 * t1;
    c[7] = Dct8::T0 * t1 - Dct8::T6 * t2;
  }
  {
    double t1 = c[2] + c[6], t2 = c[2] - c[6];
    c[2] = Dct8::T1 * t2 + Dct8::T5 * t1;
    c[6] = Dct8::T1 * t1 - Dct8::T5 * t2;
  }
  {
    double t1 = c[3] + c[5], t2 = c[3] - c[5];
    c[3] = Dct8::T2 * t2 + Dct8::T4 * t1;
    c[5] = Dct8::T2 * t1 - Dct8::T4 * t2;
  }
  c[4] = c[4] * Dct8::TWO_T3;
  rfft8_forward(c);
  if (kScale) {
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = c[k] * fct;
  }
#pragma unroll
  for (int k = 1; k < 7; k += 2) {
    double lo = c[k];
    c[k] = lo - c[k + 1];
    c[k + 1] = c[k + 1] + lo;
  }
}

}  // namespace sst
