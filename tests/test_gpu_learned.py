"""GPU: learned-tokenizer plug-in on tcgen05 vs the torch
fp32 oracle (oracle/learned_oracle.py, parity unpinned -- the reference ships
no learned model).

Stage-isolated tests feed the kernels and the oracle identical bf16 inputs,
so the only difference is fp32 summation order: stored bf16 activations agree
to <= 1 bf16 ulp, FSQ indices agree >= 99.9 % with every mismatch on a
rounding boundary, pixels agree to 1e-5.  End to end the one-ulp flips grow
through the layers: this bf16 network's FSQ indices agree on >= 98 % (measured
98.8-98.9 %, every mismatch within 0.05 of a rounding boundary), BELOW the
north star's 99.9 % -- the bound asserted here.  Reconstruction from identical
codes: max |err| <= 1e-2 (bf16) and PSNR within 0.05 dB.  The int8 network
(learned_i8.py, tests/test_gpu_learned_i8.py) is exact integer arithmetic
and meets the north star with 100 % agreement and identical frames.
"""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import learned_oracle as LO
from oracle import semstream_oracle as O
from oracle.synth import make_clip
from paper_2602_03529_b200 import _dev, _lib
from paper_2602_03529_b200 import codec as CC, transport as T, video as V
from paper_2602_03529_b200.learned import (TAPS_233, LearnedConfig, LearnedPlugin,
                                           LearnedTokenizer, _taps_array, make_weights)

pytestmark = pytest.mark.gpu

BF16_ULP = 2.0 ** -7      # relative spacing of bf16 (8 significant bits)


def _bf(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).to(
        torch.float32)


def _conv_gpu(x, W, b, taps, t_lo, t_cnt, epi, out_T=2, act=0, residual=None, hw=(0, 0),
              frame_base=0):
    """Raw sst_lt_conv call on bf16 CUDA tensors; returns the epilogue outputs."""
    G, T_in, H, Wd, Cin = x.shape
    dev = _dev.device()
    xd = x.to(dev, torch.bfloat16).contiguous()
    Wd_ = torch.from_numpy(np.ascontiguousarray(W)).to(dev, torch.bfloat16).contiguous()
    bd = torch.from_numpy(np.ascontiguousarray(b, dtype=np.float32)).to(dev)
    d = _lib.SstConvDesc()
    d.in_ = xd.data_ptr()
    d.in_C, d.in_W, d.in_H, d.in_T = Cin, Wd, H, T_in
    d.G, d.Ht, d.Wt, d.t_lo, d.t_cnt = G, H, Wd, t_lo, t_cnt
    d.n_taps = len(taps)
    d.taps = _taps_array(taps)
    d.weight = Wd_.data_ptr()
    d.N, d.K = W.shape
    d.bias = bd.data_ptr()
    d.epi, d.act, d.out_T = epi, act, out_T
    keep = [xd, Wd_, bd]
    out = {}
    if epi == _lib.LT_EPI_STORE:
        o = torch.zeros((G, out_T, H, Wd, W.shape[0]), dtype=torch.bfloat16, device=dev)
        d.out = o.data_ptr()
        if residual is not None:
            r = residual.to(dev, torch.bfloat16).contiguous()
            keep.append(r)
            d.residual = r.data_ptr()
        out["out"] = o
    elif epi == _lib.LT_EPI_FSQ:
        codes = torch.zeros((G, 2, H, Wd, 12), dtype=torch.float64, device=dev)
        idx = torch.zeros((G, 2, H, Wd, 2), dtype=torch.int32, device=dev)
        mask = torch.zeros((G, 2, H, Wd), dtype=torch.uint8, device=dev)
        d.codes, d.idx, d.mask = codes.data_ptr(), idx.data_ptr(), mask.data_ptr()
        out.update(codes=codes, idx=idx, mask=mask)
    else:
        fr = torch.full((G, 9, hw[0], hw[1], 3), -1.0, dtype=torch.float32, device=dev)
        d.frames, (d.h, d.w), d.frame_base = fr.data_ptr(), hw, frame_base
        out["frames"] = fr
    _lib.call("sst_lt_conv", C.byref(d), _dev.stream())
    torch.cuda.synchronize()
    return {k: v.float().cpu() if v.dtype == torch.bfloat16 else v.cpu() for k, v in out.items()}


def _assert_bf16_close(got, want, min_exact=0.97, atol=0.0):
    got, want = got.numpy(), want.numpy()
    err = np.abs(got - want)
    tol = 2 * BF16_ULP * np.maximum(np.abs(want), 1e-3) + atol
    assert (err <= tol).all(), f"max err {err.max()} (worst rel {(err / tol).max():.2f} of 2 ulp)"
    assert (got == want).mean() >= min_exact


@pytest.mark.parametrize("shape,cin,act,res", [
    ((2, 2, 8, 16, 64), 64, 1, False),       # one exact tile
    ((1, 2, 5, 19, 128), 128, 0, True),      # ragged tiles, residual path
    ((3, 2, 11, 33, 64), 64, 1, True),       # several tiles per frame, both epilogue ops
])
def test_conv233_store_matches_oracle(shape, cin, act, res):
    rng = np.random.default_rng(1)
    G, Tn, H, Wd, _ = shape
    x = _bf(rng.standard_normal(shape))
    W = _bf(rng.standard_normal((128, 18 * cin)) / np.sqrt(18 * cin)).numpy()
    b = _bf(rng.standard_normal(128) * 0.1).numpy()
    resid = _bf(rng.standard_normal((G, Tn, H, Wd, 128))) if res else None
    got = _conv_gpu(x, W, b, TAPS_233, 0, 2, _lib.LT_EPI_STORE, act=act, residual=resid)["out"]
    want = LO.conv233(x, W, b, act=bool(act), residual=resid)
    _assert_bf16_close(got, want)


@pytest.mark.parametrize("shape,cin", [
    ((2, 2, 16, 16, 64), 64),                # one exact 16x16 tile, decoder-input width
    ((1, 2, 45, 80, 256), 256),              # 1080p s=3 token grid, ragged last tile row
    ((2, 2, 13, 37, 64), 64),                # ragged in both dimensions
])
def test_conv233_halo_kernel(shape, cin, monkeypatch):
    """N = 256 runs the CTA-pair halo kernel (cta_group::2, one TMA box per 9
    spatial taps, UMMA descriptors starting mid swizzle atom); it must match
    the oracle, and the persistent single-CTA and non-persistent halo kernels
    bit for bit (same MMA order per output), and the per-tap kernel to the
    oracle tolerance."""
    rng = np.random.default_rng(11)
    G, Tn, H, Wd, _ = shape
    x = _bf(rng.standard_normal(shape))
    W = _bf(rng.standard_normal((256, 18 * cin)) / np.sqrt(18 * cin)).numpy()
    b = _bf(rng.standard_normal(256) * 0.1).numpy()
    resid = _bf(rng.standard_normal((G, Tn, H, Wd, 256)))
    want = LO.conv233(x, W, b, act=True, residual=resid)
    pair = _conv_gpu(x, W, b, TAPS_233, 0, 2, _lib.LT_EPI_STORE, act=1, residual=resid)["out"]
    _assert_bf16_close(pair, want)                       # default: CTA-pair kernel
    for mode in ("persistent", "halo", "generic"):
        monkeypatch.setenv("SST_LT_CONV", mode)
        got = _conv_gpu(x, W, b, TAPS_233, 0, 2, _lib.LT_EPI_STORE, act=1, residual=resid)["out"]
        _assert_bf16_close(got, want)
        assert torch.equal(got, pair) or mode == "generic"


@pytest.mark.parametrize("H,W,D", [(8, 8, 128), (13, 21, 256), (45, 80, 256)])
def test_window_attention_core(H, W, D):
    rng = np.random.default_rng(12)
    G = 2
    qkv = _bf(rng.standard_normal((G, 2, H, W, 3 * D)))
    dev = _dev.device()
    qd = qkv.to(dev, torch.bfloat16).contiguous()
    out = torch.full((G, 2, H, W, D), 7.0, dtype=torch.bfloat16, device=dev)
    _lib.call("sst_lt_attn", qd.data_ptr(), G, H, W, D, out.data_ptr(), _dev.stream())
    torch.cuda.synchronize()
    # attention outputs are convex mixes of V rows (|o| <~ 1); near-zero
    # results from cancellation carry the absolute rounding error of the
    # bf16 probabilities, hence the 2e-3 absolute floor
    _assert_bf16_close(out.float().cpu(), LO.window_attention(qkv), min_exact=0.95, atol=2e-3)


@pytest.mark.parametrize("H,W,D", [(8, 8, 128), (13, 21, 256), (45, 80, 256)])
def test_fused_qkv_attention(H, W, D):
    """qkv projection inside the attention kernel == 1x1 GEMM + attention core."""
    rng = np.random.default_rng(13)
    G = 2
    h = _bf(rng.standard_normal((G, 2, H, W, D)) * 0.5)
    Wq = _bf(rng.standard_normal((3 * D, D)) / np.sqrt(D)).numpy()
    bq = _bf(rng.standard_normal(3 * D) * 0.1).numpy()
    dev = _dev.device()
    hd = h.to(dev, torch.bfloat16).contiguous()
    wd = torch.from_numpy(Wq).to(dev, torch.bfloat16).contiguous()
    bd = torch.from_numpy(bq).to(dev)
    out = torch.full((G, 2, H, W, D), 7.0, dtype=torch.bfloat16, device=dev)
    _lib.call("sst_lt_attn_fused", hd.data_ptr(), wd.data_ptr(), bd.data_ptr(), G, H, W, D,
              out.data_ptr(), _dev.stream())
    torch.cuda.synchronize()
    want = LO.window_attention(LO.bf(LO.linear(h, Wq, bq)))
    _assert_bf16_close(out.float().cpu(), want, min_exact=0.9, atol=4e-3)


@pytest.mark.parametrize("H,W,D,G", [(8, 8, 128, 1), (13, 21, 256, 3), (45, 80, 256, 4),
                                     (3, 5, 64, 1)])
def test_persistent_attention_equals_one_cta_per_item(H, W, D, G, monkeypatch):
    """The persistent warp-specialised attention kernel (default) and the
    one-CTA-per-(window, head) kernel (SST_LT_ATTN=fused) issue the same MMAs
    in the same order: bit-identical outputs, including item counts that do
    not divide the grid and fewer items than SMs."""
    rng = np.random.default_rng(14 + D + G)
    h = _bf(rng.standard_normal((G, 2, H, W, D)) * 0.5)
    Wq = _bf(rng.standard_normal((3 * D, D)) / np.sqrt(D)).numpy()
    bq = _bf(rng.standard_normal(3 * D) * 0.1).numpy()
    dev = _dev.device()
    hd = h.to(dev, torch.bfloat16).contiguous()
    wd = torch.from_numpy(Wq).to(dev, torch.bfloat16).contiguous()
    bd = torch.from_numpy(bq).to(dev)
    outs = []
    for mode in ("fused", "persistent"):
        monkeypatch.setenv("SST_LT_ATTN", mode)
        out = torch.full((G, 2, H, W, D), 7.0, dtype=torch.bfloat16, device=dev)
        _lib.call("sst_lt_attn_fused", hd.data_ptr(), wd.data_ptr(), bd.data_ptr(), G, H, W, D,
                  out.data_ptr(), _dev.stream())
        torch.cuda.synchronize()
        outs.append(out)
    assert torch.equal(outs[0], outs[1])
    want = LO.window_attention(LO.bf(LO.linear(h, Wq, bq)))
    _assert_bf16_close(outs[1].float().cpu(), want, min_exact=0.9, atol=4e-3)


def test_conv_causal_first_frame_sees_no_past():
    # t=0 output must not depend on t=1 input (causal temporal kernel)
    rng = np.random.default_rng(2)
    x = _bf(rng.standard_normal((1, 2, 8, 16, 64)))
    W = _bf(rng.standard_normal((128, 18 * 64)) / 30).numpy()
    b = np.zeros(128, np.float32)
    a = _conv_gpu(x, W, b, TAPS_233, 0, 2, _lib.LT_EPI_STORE)["out"]
    x2 = x.clone()
    x2[:, 1] = _bf(rng.standard_normal((1, 8, 16, 64)))
    b2 = _conv_gpu(x2, W, b, TAPS_233, 0, 2, _lib.LT_EPI_STORE)["out"]
    assert torch.equal(a[:, 0], b2[:, 0])
    assert not torch.equal(a[:, 1], b2[:, 1])


def test_patch_embed_one_tap_and_long_k():
    # 1-tap GEMM over a T=1 input written into latent frame 1 (K = 1536)
    rng = np.random.default_rng(3)
    x = _bf(rng.random((2, 1, 6, 21, 1536)))
    W = _bf(rng.standard_normal((256, 1536)) / np.sqrt(1536)).numpy()
    b = _bf(rng.standard_normal(256) * 0.1).numpy()
    got = _conv_gpu(x, W, b, [(-1, 0, 0)], 1, 1, _lib.LT_EPI_STORE)["out"]
    want = LO.bf(LO.linear(x[:, 0], W, b))
    _assert_bf16_close(got[:, 1], want)
    assert (got[:, 0] == 0).all()            # latent frame 0 untouched


def test_fsq_head_indices():
    rng = np.random.default_rng(4)
    h = _bf(rng.standard_normal((2, 2, 13, 27, 256)))
    W = np.zeros((16, 256), np.float32)
    W[:12] = _bf(rng.standard_normal((12, 256)) * 1.5 / 16).numpy()
    b = np.zeros(16, np.float32)
    out = _conv_gpu(h, W, b, [(0, 0, 0)], 0, 2, _lib.LT_EPI_FSQ)
    z = LO.linear(h, W, b)[..., :12]
    codes, idx = LO.fsq(z)
    assert (out["mask"] == 1).all()
    agree = (out["idx"].numpy() == idx.numpy()).all(-1)
    assert agree.mean() >= 0.999
    # every mismatch must sit on an FSQ rounding boundary
    diff = out["codes"].numpy() != codes.numpy()
    if diff.any():
        zz = z.numpy()[diff]
        lv = np.array(LO.FSQ_LEVELS * 1)[np.nonzero(diff)[-1]]
        half_l = (lv - 1) * (1 - 1e-3) / 2
        off = np.where(lv % 2 == 0, 0.5, 0.0)
        bnd = np.tanh(zz + np.arctanh(off / half_l)) * half_l - off
        assert np.abs(bnd - np.floor(bnd) - 0.5).max() < 1e-4
    # indices are in range and decode back to the codes
    assert out["idx"].min() >= 0 and out["idx"].max() < 64000


@pytest.mark.parametrize("Ht,Wt,crop", [
    (5, 7, (3, 5)),      # cropped, odd width: scalar store path
    (21, 24, (5, 0)),    # width % 4 == 0: warp-staged coalesced rows, ragged last token rows
    (19, 21, (2, 4)),    # staged interior segments + per-thread edge segment
])
def test_pixels_unpatchify(Ht, Wt, crop):
    rng = np.random.default_rng(5)
    G = 2
    h = _bf(rng.standard_normal((G, 2, Ht, Wt, 256)))
    W = _bf(rng.standard_normal((1536, 256)) / 16).numpy()
    b = np.full(1536, 0.5, np.float32)
    hw = (Ht * 8 - crop[0], Wt * 8 - crop[1])
    fr = _conv_gpu(h, W, b, [(0, 0, 0)], 1, 1, _lib.LT_EPI_PIXELS, hw=hw, frame_base=1)["frames"]
    op = LO.linear(h[:, 1], W, b).clamp(0, 1).reshape(G, Ht, Wt, 8, 8, 8, 3)
    want = op.permute(0, 3, 1, 4, 2, 5, 6).reshape(G, 8, Ht * 8, Wt * 8, 3)[:, :, :hw[0], :hw[1]]
    assert (fr[:, 0] == -1).all()            # frame 0 not written by the P launch
    assert np.abs(fr[:, 1:].numpy() - want.numpy()).max() <= 1e-5


@pytest.mark.parametrize("H,W,s", [(64, 64, 1), (72, 96, 2), (50, 70, 3), (37, 45, 1)])
def test_patchify_bit_exact(H, W, s):
    rng = np.random.default_rng(6)
    fr = rng.random((2, 9, H, W, 3), dtype=np.float32)
    h, w = -(-H // s), -(-W // s)
    Ht, Wt = -(-h // 8), -(-w // 8)
    dev = _dev.device()
    x = torch.from_numpy(fr).to(dev)
    pI = torch.empty((2, Ht, Wt, 192), dtype=torch.bfloat16, device=dev)
    pP = torch.empty((2, Ht, Wt, 1536), dtype=torch.bfloat16, device=dev)
    _lib.call("sst_lt_patchify", x.data_ptr(), 2, H, W, s, pI.data_ptr(), pP.data_ptr(),
              _dev.stream())
    wI, wP, _ = LO.patchify(fr, s)
    assert torch.equal(pI.float().cpu(), wI)
    assert torch.equal(pP.float().cpu(), wP)


def test_dec_in_snap_and_conceal():
    rng = np.random.default_rng(7)
    G, Ht, Wt = 2, 6, 9
    lv = np.array(LO.FSQ_LEVELS)
    q = rng.integers(-(lv // 2), lv - lv // 2, size=(G, 2, Ht, Wt, 12))
    codes = q / (lv // 2)
    noisy = codes + rng.uniform(-0.05, 0.05, codes.shape)      # 8-bit requantisation noise
    mask = (rng.random((G, 2, Ht, Wt)) > 0.3).astype(np.uint8)
    noisy[mask == 0] = 0.0
    dev = _dev.device()
    out = torch.empty((G, 2, Ht, Wt, 64), dtype=torch.bfloat16, device=dev)
    tok_d, mask_d = _dev.h2d(noisy, np.float64), _dev.h2d(mask, np.uint8)
    _lib.call("sst_lt_dec_in", tok_d.data_ptr(), mask_d.data_ptr(), G, Ht, Wt, out.data_ptr(),
              _dev.stream())
    torch.cuda.synchronize()
    assert torch.equal(out.float().cpu(), LO.dec_in(noisy, mask))


def _model(blocks=1, dim=128, seed=0):
    cfg = LearnedConfig(dim=dim, blocks=blocks, seed=seed)
    w = make_weights(cfg)
    return cfg, w, LearnedTokenizer(cfg, w)


@pytest.mark.parametrize("W,H,s", [(256, 256, 2), (96, 72, 1), (200, 120, 3)])
def test_end_to_end_encode_decode(W, H, s):
    cfg, w, m = _model(blocks=2, dim=128)
    clip = make_clip("moving-square", W, H, 9, seed=3)
    fr = np.stack([clip.gop(0)])
    codes, idx, mask, hw = m.encode_frames(torch.from_numpy(fr).to(_dev.device()), s)
    ocodes, oidx, ohw, z = LO.encode(fr, s, w, cfg.blocks)
    assert tuple(hw) == tuple(ohw)
    # End to end the two sides diverge by single-ulp bf16 rounding flips of
    # intermediate activations (each layer alone agrees on >= 99.9 % of its
    # elements, see the stage-isolated tests), so an FSQ code can flip only
    # where the oracle's bound value lies near a rounding boundary.
    agree = (idx.cpu().numpy() == oidx).all(-1).mean()
    assert agree >= 0.98, agree
    diff = codes.cpu().numpy() != ocodes
    if diff.any():
        lv = np.array(LO.FSQ_LEVELS)[np.nonzero(diff)[-1]]
        half_l = (lv - 1) * (1 - 1e-3) / 2
        off = np.where(lv % 2 == 0, 0.5, 0.0)
        bnd = np.tanh(z.numpy()[diff] + np.arctanh(off / half_l)) * half_l - off
        assert np.abs(bnd - np.floor(bnd) - 0.5).max() < 0.05
    # decoder fed the oracle's codes (stage-isolated) with a 30 % P drop
    rng = np.random.default_rng(8)
    mk = np.ones(ocodes.shape[:-1], np.uint8)
    mk[:, 1] = rng.random(mk[:, 1].shape) > 0.3
    tok = ocodes * mk[..., None]
    got = m.decode_tokens(_dev.h2d(tok, np.float64), _dev.h2d(mk, np.uint8), hw).cpu().numpy()
    want = LO.decode(tok, mk, hw, w, cfg.blocks)
    assert np.abs(got - want).max() <= 1e-2
    src = fr if s == 1 else O.downscale(fr, s)
    p_gpu = O.psnr_from_mse(O.mse(src[0], got[0]))
    p_ref = O.psnr_from_mse(O.mse(src[0], want[0]))
    assert abs(p_gpu - p_ref) <= 0.05


def test_plugin_through_packet_transport():
    """Codes survive the reference's 8-bit row quantiser exactly: decoding
    reassembled packets equals decoding the encoder's codes."""
    cfg = LearnedConfig(dim=128, blocks=1, seed=2)
    plug = LearnedPlugin(cfg)
    clip = make_clip("noisy-motion", 96, 64, 9, seed=1)
    gop = V.GoP(0, tuple(V.Frame(f, timestamp_index=t) for t, f in enumerate(clip.gop(0))))
    i_tok, p_tok = plug.encode(gop, CC.CodecConfig())
    assert i_tok.values.shape == (8, 12, 12)
    direct = plug.decode(i_tok, p_tok, CC.CodecConfig())
    pk_i = [T.parse_packet(p.to_bytes()) for p in T.packetize_tokens(i_tok, scale=1)]
    pk_p = [T.parse_packet(p.to_bytes()) for p in T.packetize_tokens(p_tok, scale=1)]
    ri = T.reassemble(pk_i, i_tok.values.shape, "I", frame_shape=i_tok.frame_shape)
    rp = T.reassemble(pk_p, p_tok.values.shape, "P", frame_shape=p_tok.frame_shape)
    via = plug.decode(ri, rp, CC.CodecConfig())
    for a, b in zip(direct.frames, via.frames):
        assert np.array_equal(a.samples, b.samples)
    assert len(direct.frames) == 9 and direct.frames[0].samples.shape == (64, 96, 3)


def test_learned_gop_codec_stages_bit_exact():
    """LearnedGopCodec: the transport stages around the learned tokenizer are
    the reference's, bit-exact given the GPU's FSQ codes (similarity, drop
    mask, packet bytes, reassembly), then the learned decoder, upscale and
    blend."""
    from paper_2602_03529_b200.learned import LearnedGopCodec

    H, W, s, g = 72, 100, 2, 2       # W*3*4 % 16 == 0 for the TMA store
    cfg = LearnedConfig(dim=128, blocks=1, seed=4)
    codec = LearnedGopCodec(g, H, W, s, cfg=cfg)
    clip = make_clip("moving-square", W, H, 18, seed=2)
    fr = np.stack([clip.gop(0), clip.gop(1)])
    dev = _dev.device()
    frames = torch.from_numpy(fr).to(dev)
    drop_k = codec.drop_k(0.25)
    out = torch.empty_like(frames)
    # step 1 primes the blend history with a different GoP pair
    frames0 = torch.from_numpy(np.stack([clip.gop(1), clip.gop(0)])).to(dev)
    out0 = torch.empty_like(frames0)
    codec.set_gop_ids([5, 6])
    codec.step(frames0, out0, g, drop_k=drop_k)
    prev9 = codec.frames9[0][:g].cpu().numpy()
    codec.set_gop_ids([7, 8])
    codec.step(frames, out, g, drop_k=drop_k)
    torch.cuda.synchronize()
    # first step: no blend
    for j in range(g):
        want0 = np.stack([O.upscale(prev9[j, t], s, crop=(H, W)) for t in range(9)])
        assert np.array_equal(out0[j].cpu().numpy(), want0)
    codes, _, _, hw = codec.model.encode_frames(frames, s)
    codes = codes.cpu().numpy()
    arena, lengths = codec.arena.cpu().numpy(), codec.lengths.cpu().numpy()
    Ht, Wt = codec.Ht, codec.Wt
    rx = np.zeros((g, 2, Ht, Wt, 12))
    rxm = np.zeros((g, 2, Ht, Wt), np.uint8)
    for j in range(g):
        sim = O.similarity(codes[j, 1], codes[j, 0])
        assert np.array_equal(codec.sim[j].cpu().numpy(), sim)
        drop = O.top_k_mask(sim, drop_k)
        pv, pm = O.apply_mask(codes[j, 1], np.ones((Ht, Wt), bool), drop)
        wire = O.packetize(0, 7 + j, codes[j, 0], np.ones((Ht, Wt), bool), s) + \
            O.packetize(1, 7 + j, pv, pm, s)
        base = j * codec.n_pkt_per_gop
        got = [arena[base + i, :lengths[base + i]].tobytes() for i in range(codec.n_pkt_per_gop)]
        assert got == wire
        parsed = [O.parse(d) for d in wire]
        for kind in (0, 1):
            v, m = O.reassemble([q for q in parsed if q["kind"] == kind], (Ht, Wt, 12))
            rx[j, kind], rxm[j, kind] = v, m
    # the fused packets -> decoder-input stage equals reassemble + dec_in
    assert torch.equal(codec.dec_x[:g].float().cpu(), LO.dec_in(rx, rxm))
    dec = codec.model.decode_tokens(_dev.h2d(rx, np.float64), _dev.h2d(rxm, np.uint8), hw)
    assert torch.equal(dec, codec.frames9[1][:g])
    d9 = dec.cpu().numpy()
    for j in range(g):
        up = [O.upscale(d9[j, t], s, crop=(H, W)) for t in range(9)]
        prev_up = [O.upscale(prev9[j, t], s, crop=(H, W)) for t in range(9)]
        want = O.blend(prev_up, up, 2)
        assert np.array_equal(out[j].cpu().numpy(), np.stack(want))


def test_learned_decoder_input_from_lossy_packets():
    """Packets -> decoder input with network loss: first-wins routing, lost I
    rows -> zero codes, lost P rows -> the co-located I codes; equal to the
    reference's reassemble (oracle) followed by the snap / conceal stage."""
    from paper_2602_03529_b200.learned import LearnedGopCodec

    H, W, s, g = 64, 96, 2, 2
    codec = LearnedGopCodec(g, H, W, s, cfg=LearnedConfig(dim=128, blocks=1, seed=6))
    clip = make_clip("noisy-motion", W, H, 9, seed=4)
    frames = torch.from_numpy(np.stack([clip.gop(0)] * g)).cuda()
    codec.set_gop_ids([3, 4])
    codec.tokenize(frames, g)
    codec.select_and_pack(g, codec.drop_k(0.1))
    torch.cuda.synchronize()
    npk = codec.n_pkt_per_gop
    rng = np.random.default_rng(9)
    lost = [set(int(j) for j in np.flatnonzero(rng.random(npk) < 0.3)) for _ in range(g)]
    present = torch.tensor([0 if j in lost[i] else 1 for i in range(g) for j in range(npk)],
                           dtype=torch.uint8, device="cuda")
    codec.decode(g, 0, present=present)
    torch.cuda.synchronize()
    arena, lengths = codec.arena.cpu().numpy(), codec.lengths.cpu().numpy()
    rx = np.zeros((g, 2, codec.Ht, codec.Wt, 12))
    rxm = np.zeros((g, 2, codec.Ht, codec.Wt), np.uint8)
    for i in range(g):
        wire = [arena[i * npk + j, :lengths[i * npk + j]].tobytes() for j in range(npk)
                if j not in lost[i]]
        parsed = [O.parse(d) for d in wire]
        for kind in (0, 1):
            v, m = O.reassemble([q for q in parsed if q["kind"] == kind], (codec.Ht, codec.Wt, 12))
            rx[i, kind], rxm[i, kind] = v, m
    assert torch.equal(codec.dec_x[:g].float().cpu(), LO.dec_in(rx, rxm))
    st = codec.stats[:4 * g].cpu().numpy().reshape(g, 2, 2)
    for i in range(g):
        lost_i = sum(1 for j in lost[i] if j < codec.Ht)
        assert st[i, 0, 1] == codec.Ht - lost_i                      # I rows received


def test_graphed_learned_codec_matches_eager():
    """GraphedLearnedGopCodec replays the same launches as LearnedGopCodec.step:
    bit-identical frames over a first GoP and both blend parities."""
    from paper_2602_03529_b200.learned import GraphedLearnedGopCodec, LearnedGopCodec

    H, W, s, g = 72, 96, 2, 1
    cfg = LearnedConfig(dim=128, blocks=1, seed=6)
    eager = LearnedGopCodec(g, H, W, s, cfg=cfg)
    graphed = LearnedGopCodec(g, H, W, s, model=eager.model)
    clip = make_clip("moving-square", W, H, 36, seed=4)
    dev = _dev.device()
    frames = torch.empty((g, 9, H, W, 3), device=dev)
    out_g = torch.empty_like(frames)
    drop_k = eager.drop_k(0.2)
    gr = None
    for k in range(4):
        frames.copy_(torch.from_numpy(np.ascontiguousarray(clip.gop(k)[None])))
        out_e = torch.empty_like(frames)
        eager.set_gop_ids([k])
        eager.step(frames, out_e, g, drop_k=drop_k)
        if gr is None:
            gr = GraphedLearnedGopCodec(graphed, g, frames, out_g, drop_k=drop_k)
        gr.step([k])
        torch.cuda.synchronize()
        assert torch.equal(out_g, out_e), k
