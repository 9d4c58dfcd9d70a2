"""GPU: K5-9 (sst_upscale_blend9, the learned path's reconstruction) bit-exact
against the oracle's upscale (codec.py:217-266) + blend_boundary
(codec.py:278-296) across scales, ragged crops, both window-load paths (TMA
when w*3*4 % 16 == 0, cp.async otherwise), blend widths 1..4 and a previous
GoP at a different scale."""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import semstream_oracle as O
from paper_2602_03529_b200 import _dev, _lib

pytestmark = pytest.mark.gpu


def _run(img, s, H, W, prev=None, n=2):
    """img [G][9][h][w][3] float32 >= 0; prev: list of (frames9 [9][h'][w'][3], s')."""
    G, _, h, w, _ = img.shape
    dev = _dev.device()
    x = torch.from_numpy(img).to(dev)
    out = torch.full((G, 9, H, W, 3), -7.0, device=dev)
    keep = []
    pd_ptr = None
    if prev is not None:
        d = np.zeros(G, dtype=_lib.PREV_DTYPE)
        for g, (p9, ps) in enumerate(prev):
            t = torch.from_numpy(np.ascontiguousarray(p9)).to(dev)
            keep.append(t)
            d[g]["p_img"] = t.data_ptr()
            d[g]["h"], d[g]["w"], d[g]["s"] = p9.shape[1], p9.shape[2], ps
        pd = torch.from_numpy(d.view(np.uint8).copy()).to(dev)
        keep.append(pd)
        pd_ptr = pd.data_ptr()
    _lib.call("sst_upscale_blend9", x.data_ptr(), G, h, w, s, H, W, pd_ptr, n, out.data_ptr(),
              _dev.stream())
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _want(img9, s, H, W, prev=None, n=2):
    up = [O.upscale(img9[t], s, crop=(H, W)) for t in range(9)]
    if prev is None:
        return np.stack(up)
    p9, ps = prev
    return np.stack(O.blend([O.upscale(p9[t], ps, crop=(H, W)) for t in range(9)], up, n))


def _frames(rng, G, h, w, hi=1.0):
    x = rng.random((G, 9, h, w, 3), dtype=np.float32) * np.float32(hi)
    x[..., 0, 0, :] = 1.0          # exact extremes
    x[..., -1, -1, :] = 0.0
    return x


@pytest.mark.parametrize("H,W,s", [(50, 96, 3), (72, 100, 2), (64, 200, 2), (40, 88, 3),
                                   (33, 517, 3)])
def test_upscale9_no_prev(H, W, s):
    rng = np.random.default_rng(H * W + s)
    h, w = -(-H // s), -(-W // s)
    img = _frames(rng, 2, h, w, hi=1.3)          # > 1 exercises the clip
    got = _run(img, s, H, W)
    for g in range(2):
        assert np.array_equal(got[g], _want(img[g], s, H, W))


@pytest.mark.parametrize("n", [1, 2, 3, 4])
@pytest.mark.parametrize("H,W,s", [(50, 96, 3), (72, 100, 2)])
def test_upscale9_blend(H, W, s, n):
    rng = np.random.default_rng(7 * n + s)
    h, w = -(-H // s), -(-W // s)
    img = _frames(rng, 2, h, w)
    prev = [(_frames(rng, 1, h, w)[0], s) for _ in range(2)]
    got = _run(img, s, H, W, prev, n)
    for g in range(2):
        assert np.array_equal(got[g], _want(img[g], s, H, W, prev[g], n))


def test_upscale9_prev_at_other_scale_and_mixed_table():
    """Previous GoP at s'=2 under a current s=3 GoP, and a null entry (first
    GoP of its stream: no blend) in the same launch."""
    H, W = 48, 64
    rng = np.random.default_rng(11)
    img = _frames(rng, 2, 16, 22)
    p0 = (_frames(rng, 1, 24, 32)[0], 2)
    got = _run(img, 3, H, W, [p0, p0], 2)
    assert np.array_equal(got[0], _want(img[0], 3, H, W, p0, 2))
    # null prev for GoP 1 via a table whose second entry is empty
    dev = _dev.device()
    d = np.zeros(2, dtype=_lib.PREV_DTYPE)
    t = torch.from_numpy(p0[0]).to(dev)
    d[0]["p_img"], d[0]["h"], d[0]["w"], d[0]["s"] = t.data_ptr(), 24, 32, 2
    pd = torch.from_numpy(d.view(np.uint8).copy()).to(dev)
    x = torch.from_numpy(img).to(dev)
    out = torch.empty((2, 9, H, W, 3), device=dev)
    _lib.call("sst_upscale_blend9", x.data_ptr(), 2, 16, 22, 3, H, W, pd.data_ptr(), 2,
              out.data_ptr(), _dev.stream())
    o = out.cpu().numpy()
    assert np.array_equal(o[0], _want(img[0], 3, H, W, p0, 2))
    assert np.array_equal(o[1], _want(img[1], 3, H, W))


def test_upscale9_1080p_one_gop():
    H, W, s = 1080, 1920, 3
    rng = np.random.default_rng(5)
    img = _frames(rng, 1, 360, 640)
    prev = [(_frames(rng, 1, 360, 640)[0], 3)]
    got = _run(img, s, H, W, prev, 2)
    assert np.array_equal(got[0], _want(img[0], s, H, W, prev[0], 2))


@pytest.mark.parametrize("mode", ["sync", "async", "tma"])
def test_upscale9_load_modes_identical(mode, monkeypatch):
    monkeypatch.setenv("SST_K5_9", mode)
    H, W, s = 50, 96, 3
    rng = np.random.default_rng(3)
    img = _frames(rng, 2, 17, 32)
    prev = [(_frames(rng, 1, 17, 32)[0], 3) for _ in range(2)]
    got = _run(img, s, H, W, prev, 2)
    for g in range(2):
        assert np.array_equal(got[g], _want(img[g], s, H, W, prev[g], 2))


@pytest.mark.parametrize("n", [1, 2, 3])
def test_upscale9_negative_zero_samples(n):
    """-0.0 samples (allowed: >= 0) keep the reference's signs bit for bit:
    bilinear of -0.0 neighbourhoods gives -0.0, and the alpha = 0 blend frame
    turns it into +0.0 (0 * prev + cur)."""
    H, W, s = 48, 64, 2
    rng = np.random.default_rng(20 + n)
    img = _frames(rng, 1, 24, 32)
    img[0, :, :6, :8] = -0.0                   # whole bilinear neighbourhoods of -0.0
    prev = [(_frames(rng, 1, 24, 32)[0], 2)]
    prev[0][0][:, :6, :8] = 0.0
    got = _run(img, s, H, W, prev, n)[0]
    want = _want(img[0], s, H, W, prev[0], n)
    assert np.array_equal(got, want)
    assert np.array_equal(np.signbit(got), np.signbit(want))
    assert np.signbit(want).any()              # the case is exercised
