"""GPU: the fused reconstruction kernels (K5 `sst_upscale_blend`, K5-9
`sst_upscale_blend9`) on adversarial sample values, bit-exact against the
oracle's upscale (codec.py:217-245) + blend_boundary (codec.py:278-296).

The kernels evaluate two blend weights in float arithmetic instead of the
reference's float64 (alpha = 0: fmaf(0, prev, cur); alpha = 1/2:
(prev + cur) * 0.5f -- upscale.cu `blend_w`).  The argument for bit identity
covers signed zeros, subnormals and operands whose exponents are far apart;
these inputs exercise exactly those cases: whole -0.0 neighbourhoods in the
previous GoP AND the current one, subnormal and near-subnormal samples,
samples at 2^-120..2^-100 next to samples near 1, and random mantissas."""

import numpy as np
import pytest
import torch

from oracle import semstream_oracle as O
from paper_2602_03529_b200 import _dev, _lib

pytestmark = pytest.mark.gpu


def _adversarial(rng, shape):
    x = rng.random(shape, dtype=np.float32)
    kind = rng.integers(0, 8, size=shape[:-1])[..., None] * np.ones(shape, np.int64)
    tiny = np.float32(2.0) ** rng.integers(-149, -100, size=shape).astype(np.float32)
    sub = (rng.integers(1, 1 << 23, size=shape) * np.float32(2.0) ** -149).astype(np.float32)
    near1 = (np.float32(1.0) - rng.integers(1, 64, size=shape).astype(np.float32) * np.float32(2.0) ** -24)
    x = np.where(kind == 0, np.float32(-0.0), x)
    x = np.where(kind == 1, np.float32(0.0), x)
    x = np.where(kind == 2, sub, x)
    x = np.where(kind == 3, tiny, x)
    x = np.where(kind == 4, near1, x)
    x = np.where(kind == 5, np.float32(1.0), x)
    return x.astype(np.float32)


def _prev_desc(dev, ptrs, h, w, s):
    d = np.zeros(len(ptrs), dtype=_lib.PREV_DTYPE)
    d["p_img"] = np.asarray(ptrs, dtype=np.uint64)
    d["h"], d["w"], d["s"] = h, w, s
    return torch.from_numpy(d.view(np.uint8).copy()).to(dev)


# (w * 3 * 4) % 16 == 0 selects the TMA-window kernels (v2 by default), the
# others the register-staged variant; odd H / W exercise the crop
@pytest.mark.parametrize("s,H,W", [(2, 48, 64), (3, 45, 72), (2, 47, 96), (3, 40, 56), (2, 33, 90)])
@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_k5_blend_adversarial_values(s, H, W, n):
    rng = np.random.default_rng(1000 * s + 10 * n + H)
    h, w = -(-H // s), -(-W // s)
    G = 3
    img = _adversarial(rng, (G, 2, h, w, 3))            # [G][I, P][h][w][3]
    prv = _adversarial(rng, (G, h, w, 3))                # previous GoPs' P images
    img[0, :, :4, :6] = -0.0                             # -0.0 neighbourhoods on both sides
    prv[0, :4, :6] = -0.0
    img[1, :, :4, :6] = np.float32(2.0) ** -149          # smallest subnormal vs ...
    prv[1, :4, :6] = np.float32(2.0) ** -148
    dev = _dev.device()
    x = torch.from_numpy(img).to(dev)
    p = torch.from_numpy(prv).to(dev)
    pd = _prev_desc(dev, [p[g].data_ptr() for g in range(G)], h, w, s)
    out = torch.full((G, 9, H, W, 3), -7.0, device=dev)
    _lib.call("sst_upscale_blend", x.data_ptr(), G, h, w, s, H, W, pd.data_ptr(), n, out.data_ptr(),
              _dev.stream())
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    for g in range(G):
        ui = O.upscale(img[g, 0], s, crop=(H, W))
        up = O.upscale(img[g, 1], s, crop=(H, W))
        uq = O.upscale(prv[g], s, crop=(H, W))
        want = np.stack(O.blend([uq] * 9, [ui] + [up] * 8, n))
        assert np.array_equal(got[g].view(np.uint32), want.view(np.uint32)), f"GoP {g}"


@pytest.mark.parametrize("s,H,W", [(2, 48, 64), (3, 45, 72), (3, 45, 66)])
@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_k5_9_blend_adversarial_values(s, H, W, n):
    """K5-9 over float32 working frames with the same adversarial values."""
    rng = np.random.default_rng(77 + 10 * n + s)
    h, w = -(-H // s), -(-W // s)
    G = 2
    img = _adversarial(rng, (G, 9, h, w, 3))
    prv = _adversarial(rng, (G, 9, h, w, 3))
    img[0, :, :4, :6] = -0.0
    prv[0, :, :4, :6] = -0.0
    dev = _dev.device()
    x = torch.from_numpy(img).to(dev)
    p = torch.from_numpy(prv).to(dev)
    pd = _prev_desc(dev, [p[g].data_ptr() for g in range(G)], h, w, s)
    out = torch.full((G, 9, H, W, 3), -7.0, device=dev)
    _lib.call("sst_upscale_blend9", x.data_ptr(), G, h, w, s, H, W, pd.data_ptr(), n, out.data_ptr(),
              _dev.stream())
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    for g in range(G):
        up = [O.upscale(img[g, t], s, crop=(H, W)) for t in range(9)]
        uq = [O.upscale(prv[g, t], s, crop=(H, W)) for t in range(9)]
        want = np.stack(O.blend(uq, up, n))
        assert np.array_equal(got[g].view(np.uint32), want.view(np.uint32)), f"GoP {g}"
