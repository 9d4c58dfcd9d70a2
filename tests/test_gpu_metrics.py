"""GPU: the reference's parity metrics (video.py:265-322)
on the device, bit-identical to numpy: mse / gop_psnr, boundary_flicker (l1,
l2) and inter_frame_consistency reduce in numpy's pairwise summation order
(csrc/metrics.cu).  The golden-fixture PSNR / MSE of every reference GoP is
asserted in test_gpu_golden.py."""

import numpy as np
import pytest
import torch

from oracle import semstream_oracle as O
from paper_2602_03529_b200 import video as V

pytestmark = pytest.mark.gpu


def _frames(rng, n, shape):
    a = rng.random((n,) + shape) * 2.0 ** rng.integers(-30, 1, (n,) + shape)
    a[rng.random(a.shape) < 0.05] = 0.0
    a[rng.random(a.shape) < 0.03] = 1.0
    return np.clip(a, 0, 1).astype(np.float32)


SHAPES = [(1,), (7,), (8,), (9,), (127,), (128,), (129,), (136,), (1000,), (4099,),
          (37, 41, 3), (128, 128, 3), (240, 427, 3), (720, 1280, 3), (1080, 1920, 3)]


@pytest.mark.parametrize("shape", SHAPES, ids=[str(s) for s in SHAPES])
def test_mse_bit_identical_to_numpy(rng, shape):
    a, b = _frames(rng, 3, shape), _frames(rng, 3, shape)
    got = V._mean_diff(list(a), list(b), 0)
    want = [O.mse(x, y) for x, y in zip(a, b)]
    assert [float(g) for g in got] == want
    got1 = V._mean_diff(list(a), list(b), 1)
    want1 = [float(np.mean(np.abs(x.astype(np.float64) - y.astype(np.float64))))
             for x, y in zip(a, b)]
    assert [float(g) for g in got1] == want1


def test_gop_psnr_cap_and_identity(rng):
    f = _frames(rng, 9, (16, 24, 3))
    g = V.GoP(0, tuple(V.Frame(x, timestamp_index=t) for t, x in enumerate(f)))
    assert V.gop_psnr(g, g) == (99.0, 0.0)
    h = V.GoP(0, tuple(V.Frame(np.clip(x + 0.01, 0, 1).astype(np.float32), timestamp_index=t)
                       for t, x in enumerate(f)))
    assert V.gop_psnr(g, h) == O.gop_psnr(list(f), [x.samples for x in h.frames])
    with pytest.raises(ValueError):
        V.mse(V.Frame(f[0]), V.Frame(f[0][:8]))


@pytest.mark.parametrize("n", range(1, 10))
def test_flicker_and_consistency_bit_identical(rng, n):
    shape = (45, 80, 3)
    p, c = _frames(rng, 9, shape), _frames(rng, 9, shape)
    gp = V.GoP(0, tuple(V.Frame(x, timestamp_index=t) for t, x in enumerate(p)))
    gc = V.GoP(1, tuple(V.Frame(x, timestamp_index=t) for t, x in enumerate(c)))
    for norm in ("l1", "l2"):
        assert V.boundary_flicker(gp, gc, n, norm) == O.boundary_flicker(p, c, n, norm)
    assert V.inter_frame_consistency(gc.frames) == O.inter_frame_consistency(c)


def test_gop_psnr_device_matches_host(rng):
    f, g = _frames(rng, 9, (180, 320, 3)), _frames(rng, 9, (180, 320, 3))
    dev = V.gop_psnr_device(torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda())
    assert dev == O.gop_psnr(list(f), list(g))
