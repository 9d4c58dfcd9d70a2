"""ORACLE / TEST INFRASTRUCTURE ONLY -- never imported by the product path.

Bit-exact CPU restatement of the 8-point orthonormal DCT-II / DCT-III that the
reference obtains from ``scipy.fft.dctn`` / ``idctn`` (reference call sites:
``pkg/src/semstream/codec.py:123`` and ``codec.py:138``).

Third-party dependency restated here (absent from /root/reference):
  scipy 1.18.1 -> ``scipy.fft._duccfft`` (ducc0 FFT, M. Reinecke), pinned by
  ``pkg/pyproject.toml:12`` only as ``scipy>=1.10``.

Published algorithm being restated (ducc0 ``T_dcst23`` on top of the
FFTPACK-style real FFT ``rfftp``):

* DCT-II of length N=8 = FFTPACK ``cosqb``: pre-butterfly of odd/even pairs,
  a *backward* real FFT (radix-2 pass with ido=4, then radix-4 pass with
  ido=1, l1=2), a twiddle post-rotation with tw[k] = cos(pi*(k+1)/16) as
  produced by ducc0's octant-reduced ``UnityRoots(32)``, then the ortho
  correction c[0] *= sqrt2/2.
* DCT-III (the inverse) = FFTPACK ``cosqf``: ortho pre-scaling c[0] *= sqrt2,
  twiddle pre-rotation, *forward* real FFT (radix-4 pass, then radix-2),
  post-butterfly.
* ``dctn(axes=(-2,-1))`` runs the y axis first with the joint normalisation
  factor 1/sqrt(2N*2N) = 1/16 (a power of two, so where it is applied does not
  change any bit), then the x axis with factor 1.

The twiddle constants below are the exact doubles ducc0 computes (octant
symmetry: e.g. the pi/4 entry is sin(fl(pi/4)) = 0.7071067811865475, one ulp
below the correctly-rounded cos(pi/4)).  The restatement was pinned against
``scipy.fft.dct/idct/dctn/idctn`` on random inputs (tests/test_oracle_dct.py)
and is bit-identical, including signed zeros.

Every operation is a separately rounded IEEE-754 binary64 add/sub/mul; numpy
ufuncs never contract into FMA, matching the compiled ducc0 kernels.  The CUDA
kernels (paper_2602_03529_b200/csrc/dct8.cuh) implement the same sequence with
``-fmad=false``.
"""

from __future__ import annotations

import numpy as np

# ducc0 UnityRoots(32)[k+1].r for k = 0..7 (DCT twiddles)
TW = (0.9807852804032304, 0.9238795325112867, 0.8314696123025452,
      0.7071067811865475, 0.5555702330196022, 0.3826834323650898,
      0.19509032201612825, -0.0)
# ducc0 UnityRoots(8)[1] (rfft radix-2 pass twiddle, real / imag part)
W8_RE = 0.7071067811865475
W8_IM = 0.7071067811865476
SQRT2 = 1.4142135623730951
HALF_SQRT2 = SQRT2 * 0.5          # ortho DC factor of the DCT-II
TWO_TW3 = 2.0 * TW[3]             # c[N/2] factor of the DCT-III


def _split(x: np.ndarray):
    return [np.array(x[..., j], dtype=np.float64) for j in range(8)]


def _rfft_backward8(c):
    """Half-complex -> real backward FFT of length 8 (radix-2 then radix-4)."""
    # radix-2 pass, ido=4, l1=1
    d = [None] * 8
    d[0] = c[0] + c[7]
    d[4] = c[0] - c[7]
    d[3] = 2.0 * c[3]
    d[7] = -2.0 * c[4]
    d[1] = c[1] + c[5]
    tr2 = c[1] - c[5]
    ti2 = c[2] + c[6]
    d[2] = c[2] - c[6]
    d[6] = W8_RE * ti2 + W8_IM * tr2
    d[5] = W8_RE * tr2 - W8_IM * ti2
    # radix-4 pass, ido=1, l1=2
    e = [None] * 8
    for k in (0, 1):
        a0, a1, a2, a3 = d[4 * k], d[4 * k + 1], d[4 * k + 2], d[4 * k + 3]
        s03 = a0 + a3
        d03 = a0 - a3
        t1 = 2.0 * a1
        t2 = 2.0 * a2
        e[k] = s03 + t1
        e[k + 4] = s03 - t1
        e[k + 6] = d03 + t2
        e[k + 2] = d03 - t2
    return e


def _rfft_forward8(c):
    """Real -> half-complex forward FFT of length 8 (radix-4 then radix-2)."""
    # radix-4 pass, ido=1, l1=2
    d = [None] * 8
    for k in (0, 1):
        s31 = c[k + 6] + c[k + 2]
        d[4 * k + 2] = c[k + 6] - c[k + 2]
        s02 = c[k] + c[k + 4]
        d[4 * k + 1] = c[k] - c[k + 4]
        d[4 * k] = s02 + s31
        d[4 * k + 3] = s02 - s31
    # radix-2 pass, ido=4, l1=1
    e = [None] * 8
    e[0] = d[0] + d[4]
    e[7] = d[0] - d[4]
    e[4] = -d[7]
    e[3] = d[3]
    tr2 = W8_RE * d[5] + W8_IM * d[6]
    ti2 = W8_RE * d[6] - W8_IM * d[5]
    e[1] = d[1] + tr2
    e[5] = d[1] - tr2
    e[2] = ti2 + d[2]
    e[6] = ti2 - d[2]
    return e


def dct2_last(x: np.ndarray, fct: float = 0.25) -> np.ndarray:
    """Orthonormal DCT-II along the last axis (length 8), ducc0 op order.

    ``fct`` is the pocketfft/ducc0 normalisation factor: 1/4 for a 1-D ortho
    transform, 1/16 for the first axis of a 2-D one and 1 for the second.
    """
    c = _split(x)
    c[0] = c[0] * 2.0
    c[7] = c[7] * 2.0
    for k in (1, 3, 5):
        hi = c[k + 1]
        c[k + 1] = hi - c[k]
        c[k] = c[k] + hi
    c = _rfft_backward8(c)
    if fct != 1.0:
        c = [v * fct for v in c]
    for k, kc in ((1, 7), (2, 6), (3, 5)):
        t1 = TW[k - 1] * c[kc] + TW[kc - 1] * c[k]
        t2 = TW[k - 1] * c[k] - TW[kc - 1] * c[kc]
        c[k] = 0.5 * (t1 + t2)
        c[kc] = 0.5 * (t1 - t2)
    c[4] = c[4] * TW[3]
    c[0] = c[0] * HALF_SQRT2
    return np.stack(c, axis=-1)


def dct3_last(x: np.ndarray, fct: float = 0.25) -> np.ndarray:
    """Orthonormal DCT-III (inverse of ``dct2_last``) along the last axis."""
    c = _split(x)
    c[0] = c[0] * SQRT2
    for k, kc in ((1, 7), (2, 6), (3, 5)):
        t1 = c[k] + c[kc]
        t2 = c[k] - c[kc]
        c[k] = TW[k - 1] * t2 + TW[kc - 1] * t1
        c[kc] = TW[k - 1] * t1 - TW[kc - 1] * t2
    c[4] = c[4] * TWO_TW3
    c = _rfft_forward8(c)
    if fct != 1.0:
        c = [v * fct for v in c]
    for k in (1, 3, 5):
        lo = c[k]
        c[k] = lo - c[k + 1]
        c[k + 1] = c[k + 1] + lo
    return np.stack(c, axis=-1)


def dctn2_8x8(blocks: np.ndarray) -> np.ndarray:
    """``scipy.fft.dctn(blocks, type=2, norm='ortho', axes=(-2, -1))``."""
    t = dct2_last(np.swapaxes(blocks, -1, -2), fct=1.0 / 16.0)   # along y
    t = np.swapaxes(t, -1, -2)
    return dct2_last(t, fct=1.0)                                   # along x


def idctn2_8x8(coeffs: np.ndarray) -> np.ndarray:
    """``scipy.fft.idctn(coeffs, type=2, norm='ortho', axes=(-2, -1))``."""
    t = dct3_last(np.swapaxes(coeffs, -1, -2), fct=1.0 / 16.0)    # along y
    t = np.swapaxes(t, -1, -2)
    return dct3_last(t, fct=1.0)                                   # along x
