"""CPU: numerical evidence for the places where the kernels replace the
reference's float64 arithmetic by cheaper arithmetic with a written proof
(DESIGN.md §3).  Each identity is checked in numpy (IEEE round-to-nearest
float32 / float64 operations, the same as the kernels' __fadd_rn / __dmul_rn
/ ...) on millions of values chosen to stress it: signed zeros, subnormals,
exponent spreads beyond float64's reach, rounding ties.

* upscale.cu blend_w, alpha = 1/2:  float32((q + u) * 0.5)
      == float32(0.5 * float64(q) + 0.5 * float64(u))
* encode.cu k_encode_u8 / upscale.cu K5-9 table:  float32(q) / 255 * 2^32
      == q * 0x01010100 + 2^(msb(q) + 1)
* encode.cu k_encode_u8, s = 3:  float32(float64(N 2^-32) / 9)
      == float32(float64(N) * (2^-32 / 9))   for integers N < 9 * 2^32
* encode.cu k_encode_u8:  (x + c) - c,  c = 1.5 * 2^(e(x) + 29)
      == float64(float32(x))   for x = 0 or x in [2^-12, 1]
* upscale.cu rgb24_q: the float32 byte quantiser rint(float32(v * 255))
      taken from the bits of t + 1.5 * 2^23
* upscale.cu q8_check: the same byte from the exact product inside an FMA,
      valid whenever the FMA-computed distance to a tie exceeds tau
"""

import numpy as np

RNG = np.random.default_rng(20261017)


def _wide_float32(n):
    """float32 in [0, 1] with a wide exponent range: subnormals, tiny normals,
    values near 1, exact 0 / -0 / 1."""
    e = RNG.integers(-149, 1, n)
    m = RNG.random(n) + 0.5
    x = np.ldexp(m, e).astype(np.float32)
    pick = RNG.random(n)
    x = np.where(pick < 0.02, np.float32(0.0), x)
    x = np.where((pick >= 0.02) & (pick < 0.04), np.float32(-0.0), x)
    x = np.where((pick >= 0.04) & (pick < 0.06), np.float32(1.0), x)
    x = np.where((pick >= 0.06) & (pick < 0.2), RNG.random(n).astype(np.float32), x)
    return np.minimum(x, np.float32(1.0)).astype(np.float32)


def _bits(a):
    return np.asarray(a).view(np.uint32 if np.asarray(a).dtype == np.float32 else np.uint64)


def test_half_blend_in_float32():
    n = 4_000_000
    q, u = _wide_float32(n), _wide_float32(n)
    fast = (q + u) * np.float32(0.5)                                  # float32 ops
    ref = (0.5 * q.astype(np.float64) + 0.5 * u.astype(np.float64)).astype(np.float32)
    assert np.array_equal(_bits(fast), _bits(ref))


def test_q255_identity_all_bytes():
    q = np.arange(256)
    f = (q.astype(np.float32) / np.float32(255)).astype(np.float64) * 2.0 ** 32
    g = np.array([0] + [2 << (int(x).bit_length() - 1) for x in range(1, 256)])
    assert np.array_equal(f, (q * 0x01010100 + g).astype(np.float64))


def test_mean_of_nine_as_multiply():
    n = 4_000_000
    N = RNG.integers(0, 9 * 2 ** 32, n, dtype=np.int64)
    # values of the form 9 M + r around float32 tie points of N / 9 as well
    t = RNG.integers(1, 2 ** 24, n // 4, dtype=np.int64)
    sh = RNG.integers(0, 12, n // 4)
    N = np.concatenate([N, ((2 * t + 1) << sh) * 9 // 2 + RNG.integers(-2, 3, n // 4)])
    N = N[(N >= 0) & (N < 9 * 2 ** 32)]
    s = N.astype(np.float64) * 2.0 ** -32                              # exact
    ref = (s / 9.0).astype(np.float32)
    fast = (N.astype(np.float64) * (2.0 ** -32 / 9.0)).astype(np.float32)
    assert np.array_equal(_bits(ref), _bits(fast))


def test_float32_rounding_by_magic_constant():
    n = 4_000_000
    x = np.ldexp(RNG.random(n) + 0.5, RNG.integers(-12, 1, n))
    x = np.concatenate([x, [0.0, 1.0, 2.0 ** -12, 1.0 - 2.0 ** -30]])
    x = x[(x == 0) | ((x >= 2.0 ** -12) & (x <= 1.0))]
    # ties of float32 rounding: a float32 plus half its ulp
    f = RNG.random(n // 4).astype(np.float32) * np.float32(0.5) + np.float32(0.5)
    ties = f.astype(np.float64) + 2.0 ** -25
    x = np.concatenate([x, ties[ties <= 1.0]])
    hi = (x.view(np.uint64) >> np.uint64(32)).astype(np.uint64)
    c = (((hi & np.uint64(0x7FF00000)) + np.uint64(29 << 20) + np.uint64(0x00080000)) << np.uint64(32)).view(np.float64)
    fast = (x + c) - c
    ref = x.astype(np.float32).astype(np.float64)
    assert np.array_equal(_bits(fast), _bits(ref))


def test_byte_quantiser_from_magic_add():
    n = 2_000_000
    v = _wide_float32(n)
    k = RNG.integers(0, 255, n // 2)
    v = np.concatenate([v, ((2 * k + 1) / 510.0).astype(np.float32)])  # rint ties after * 255
    t = v * np.float32(255.0)                                          # float32 product
    m = t + np.float32(12582912.0)
    byte = m.view(np.uint32) & np.uint32(0xFF)
    ref = np.rint(v * 255.0).astype(np.uint8)                          # write_raw_video
    assert np.array_equal(byte.astype(np.uint8), ref)


def test_fma_byte_quantiser_outside_tie_band():
    """q8_check: m = fma(v, 255, 1.5 * 2^23) rounds the exact 255 v to an
    integer (float32 ulp 1 there); d = fma(v, 255, -(m - 1.5 * 2^23)) is one
    rounding of 255 v - rint(255 v).  Whenever |d| <= 0.5 - tau the byte is
    write_raw_video's rint(float32(v * 255)), also for v perturbed by up to
    the kernel's proven error bound (1.22e-4 / 255)."""
    tau = np.float32(1.25 * 2.0 ** -13)
    n = 2_000_000
    v = _wide_float32(n)
    k = RNG.integers(0, 255, n // 2)
    t0 = ((2 * k + 1) / 510.0).astype(np.float32)
    v = np.concatenate([v, t0, np.nextafter(t0, np.float32(0)), np.nextafter(t0, np.float32(1))])
    t = v.astype(np.float64) * 255.0                       # exact: 24 + 8 bits
    m = np.rint(t)                                         # the FMA's rounding to the integer grid
    d = (t - m).astype(np.float32)                         # exact difference, one float32 rounding
    ok = np.abs(d) <= np.float32(0.5) - tau
    byte = m.astype(np.int64) & 0xFF
    ref = np.rint(v * np.float32(255.0)).astype(np.uint8)   # write_raw_video on the float32 sample
    assert np.array_equal(byte[ok], ref[ok].astype(np.int64))
    # the reference's sample may differ from the kernel's estimate by the bound
    eps = 1.22e-4 / 255.0
    for sgn in (-1.0, 1.0):
        vr = np.clip(v.astype(np.float64) + sgn * eps, 0.0, 1.0).astype(np.float32)
        ref_r = np.rint(vr * np.float32(255.0)).astype(np.int64)
        assert np.array_equal(byte[ok], ref_r[ok])
    assert (~ok[:n]).mean() < 1e-3 and not ok[n:n + n // 2].any()   # few detours, every tie flagged
