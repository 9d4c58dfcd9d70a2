"""GPU: the raw-rgb24 boundary of the path -- the reference CLI's file formats
(load_raw_video, video.py:130-135; write_raw_video, video.py:139-143) fused
into K1 (`sst_encode_u8`) and K5 (`sst_upscale_blend_u8`).  Bit-exact against
the float32 kernels on the converted frames (themselves pinned to the oracle
and the reference) and against the oracle's pipeline followed by the
reference's quantiser, including shapes that take the unaligned load paths,
right / bottom edge replication and rint ties."""

import numpy as np
import pytest
import torch

from oracle import semstream_oracle as O
from oracle.synth import make_clip
from paper_2602_03529_b200 import _dev, _lib
from paper_2602_03529_b200.pipeline import StreamBank

pytestmark = pytest.mark.gpu


def _encode(fn, frames, s, work=True):
    G, _, H, W, _ = frames.shape
    h, w = -(-H // s), -(-W // s)
    Ht, Wt = -(-h // 8), -(-w // 8)
    dev = _dev.device()
    tok = torch.full((G, 2, Ht, Wt, 12), -5.0, dtype=torch.float64, device=dev)
    sim = torch.full((G, Ht, Wt), -5.0, dtype=torch.float64, device=dev)
    wk = torch.full((G, 9, h, w, 3), -5.0, device=dev) if work else None
    _lib.call(fn, frames.data_ptr(), G, H, W, s, tok.data_ptr(), sim.data_ptr(),
              None if wk is None else wk.data_ptr(), _dev.stream())
    torch.cuda.synchronize()
    return tok.cpu().numpy(), sim.cpu().numpy(), None if wk is None else wk.cpu().numpy()


def _bits_equal(a, b):
    return a.shape == b.shape and np.array_equal(a.view(np.uint64 if a.dtype == np.float64 else np.uint32),
                                                  b.view(np.uint64 if b.dtype == np.float64 else np.uint32))


# aligned (16-byte rows: cp.async tiles) and unaligned widths, ragged edges, every scale
@pytest.mark.parametrize("s,H,W", [(3, 48, 64), (2, 48, 64), (1, 32, 64), (3, 50, 70), (2, 37, 90),
                                   (3, 72, 160), (2, 30, 33), (1, 17, 23), (3, 1080 // 4, 1920 // 2)])
def test_encode_u8_equals_float_path(s, H, W):
    rng = np.random.default_rng(H * 1000 + W + s)
    G = 2
    raw = rng.integers(0, 256, (G, 9, H, W, 3), dtype=np.uint8)
    raw[0, :, :3, :5] = 0                                    # exact zeros and ones
    raw[1, :, -3:, -5:] = 255
    dev = _dev.device()
    t8, s8, w8 = _encode("sst_encode_u8", torch.from_numpy(raw).to(dev), s)
    tf, sf, wf = _encode("sst_encode_work", torch.from_numpy(O.frames_from_rgb24(raw)).to(dev), s)
    assert _bits_equal(t8, tf)
    assert _bits_equal(s8, sf)
    assert _bits_equal(w8, wf)


def test_encode_u8_matches_oracle_directly():
    rng = np.random.default_rng(7)
    raw = rng.integers(0, 256, (1, 9, 45, 61, 3), dtype=np.uint8)
    tok, sim, work = _encode("sst_encode_u8", torch.from_numpy(raw).to(_dev.device()), 3)
    frames = O.frames_from_rgb24(raw[0])
    wk = O.downscale(frames, 3)
    i_vals, p_vals = O.encode(wk)
    assert np.array_equal(work[0], wk)
    assert np.array_equal(tok[0, 0], i_vals) and np.array_equal(tok[0, 1], p_vals)
    assert np.array_equal(sim[0], O.similarity(p_vals, i_vals))


def _ties(rng, shape):
    """float32 samples in [0, 1]: random, exact rint ties (v * 255 = k + 1/2
    after the float32 product) and their neighbours, zeros, -0.0, ones."""
    x = rng.random(shape, dtype=np.float32)
    k = rng.integers(0, 255, shape)
    t = ((2 * k + 1) / 510.0).astype(np.float32)
    pick = rng.integers(0, 6, shape)
    x = np.where(pick == 0, t, x)
    x = np.where(pick == 1, np.nextafter(t, np.float32(0)), x)
    x = np.where(pick == 2, np.nextafter(t, np.float32(1)), x)
    x = np.where(pick == 3, np.float32(0.0), x)
    x = np.where(pick == 4, np.float32(-0.0), x)
    return np.clip(x, -0.0, 1.0).astype(np.float32)


@pytest.mark.parametrize("s,H,W", [(2, 48, 64), (3, 45, 72), (3, 40, 56), (2, 33, 91)])
@pytest.mark.parametrize("n", [1, 2, 4])
@pytest.mark.parametrize("with_prev", [False, True])
@pytest.mark.parametrize("variant", ["default", "u8f4", "v2", "band16", "band32", "band48"])
def test_upscale_blend_u8_equals_quantised_float(s, H, W, n, with_prev, variant, monkeypatch):
    if variant.startswith("band"):
        monkeypatch.setenv("SST_K5U8_BAND", variant[4:])
    elif variant != "default":
        monkeypatch.setenv("SST_K5_VARIANT", variant)
    rng = np.random.default_rng(31 * s + n + H)
    h, w = -(-H // s), -(-W // s)
    G = 3
    img = _ties(rng, (G, 2, h, w, 3))
    prv = _ties(rng, (G, h, w, 3))
    dev = _dev.device()
    x = torch.from_numpy(img).to(dev)
    p = torch.from_numpy(prv).to(dev)
    pd = None
    if with_prev:
        d = np.zeros(G, dtype=_lib.PREV_DTYPE)
        d["p_img"] = [p[g].data_ptr() for g in range(G)]
        d["h"], d["w"], d["s"] = h, w, s
        pd = torch.from_numpy(d.view(np.uint8).copy()).to(dev)
    of = torch.empty((G, 9, H, W, 3), device=dev)
    o8 = torch.full((G, 9, H, W, 3), 7, dtype=torch.uint8, device=dev)
    args = (G, h, w, s, H, W, None if pd is None else pd.data_ptr(), n)
    _lib.call("sst_upscale_blend", x.data_ptr(), *args, of.data_ptr(), _dev.stream())
    _lib.call("sst_upscale_blend_u8", x.data_ptr(), *args, o8.data_ptr(), _dev.stream())
    torch.cuda.synchronize()
    got = o8.cpu().numpy()
    assert np.array_equal(got, O.rgb24_from_frames(of.cpu().numpy()))
    # and against the oracle's own reconstruction for one GoP
    ui = O.upscale(img[0, 0], s, crop=(H, W))
    up = O.upscale(img[0, 1], s, crop=(H, W))
    want = [ui] + [up] * 8
    if with_prev:
        want = O.blend([O.upscale(prv[0], s, crop=(H, W))] * 9, want, n)
    assert np.array_equal(got[0], O.rgb24_from_frames(np.stack(want)))


@pytest.mark.parametrize("HW", [(72, 96), (60, 70)])
def test_streambank_raw_rgb24_end_to_end(HW):
    """StreamBank with raw-rgb24 frames in and out (the CLI's encode input and
    decode output) == load_raw_video -> the oracle pipeline -> write_raw_video,
    packets byte-identical, variable scale and blending across GoPs."""
    H, W = HW
    n_streams, n_gops = 3, 3
    clips = [make_clip("noisy-motion" if i % 2 else "moving-square", W, H, 9 * n_gops, seed=40 + i)
             for i in range(n_streams)]
    raws = [[O.rgb24_from_frames(c.gop(k)) for k in range(n_gops)] for c in clips]
    sched = [(3, 2, 3), (2, 2, 3), (3, 3, 2)]
    bank = StreamBank(n_streams, H, W, blend_n=2)
    prev = [None] * n_streams
    for k in range(n_gops):
        by_s = {}
        for i in range(n_streams):
            by_s.setdefault(sched[i][k], []).append(i)
        frames = {s: torch.from_numpy(np.stack([raws[i][k] for i in ids])).cuda() for s, ids in by_s.items()}
        outs = {s: torch.empty_like(f) for s, f in frames.items()}
        bank.step(frames, outs, by_s, {s: [k] * len(ids) for s, ids in by_s.items()}, drop_rate=0.2)
        torch.cuda.synchronize()
        for s, ids in by_s.items():
            codec = bank.codecs[s]
            arena = codec.arena.cpu().numpy()
            lengths = codec.lengths.cpu().numpy()
            npk = codec.n_pkt_per_gop
            got = outs[s].cpu().numpy()
            assert got.dtype == np.uint8
            for j, i in enumerate(ids):
                ref = O.pipeline_gop(O.frames_from_rgb24(raws[i][k]), s, gop_id=k, drop_rate=0.2,
                                     prev_out=prev[i], blend_width=2)
                prev[i] = ref["frames"]
                wire = [arena[j * npk + q, :lengths[j * npk + q]].tobytes() for q in range(npk)]
                assert wire == ref["wire"], (k, i)
                assert np.array_equal(got[j], O.rgb24_from_frames(np.stack(ref["frames"]))), (k, i, s)


def test_streambank_rgb24_rejects_wide_blend():
    H, W = 48, 64
    bank = StreamBank(1, H, W, blend_n=6)
    frames = torch.zeros((1, 9, H, W, 3), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(frames)
    with pytest.raises(ValueError, match="float32"):
        bank.step({3: frames}, {3: out}, {3: [0]}, {3: [0]})
