"""CPU: the learned-tokenizer oracle (oracle/learned_oracle.py) against
independent restatements and known answers, plus the host-side weight
construction (no GPU)."""

import numpy as np
import pytest
import torch

from oracle import learned_oracle as LO
from paper_2602_03529_b200.learned import (TAPS_233, LearnedConfig, make_weights,
                                           FSQ_LEVELS as PROD_LEVELS)


def _loop_conv233(x, W, b):
    """Explicit tap loop: out[t,y,x] = sum_tap W_tap . x[t+dt, y+dy, x+dx] (zero outside)."""
    G, T, H, Wd, C = x.shape
    N = W.shape[0]
    out = np.zeros((G, T, H, Wd, N), np.float64)
    Wt = W.reshape(N, len(TAPS_233), C)
    xp = np.zeros((G, T + 1, H + 2, Wd + 2, C))
    xp[:, 1:, 1:-1, 1:-1] = x
    for k, (dt, dy, dx) in enumerate(TAPS_233):
        sl = xp[:, 1 + dt:1 + dt + T, 1 + dy:1 + dy + H, 1 + dx:1 + dx + Wd]
        out += sl @ Wt[:, k].T.astype(np.float64)
    return out + b


def test_conv233_matches_explicit_tap_loop():
    rng = np.random.default_rng(0)
    x = LO.bf(torch.from_numpy(rng.standard_normal((2, 2, 5, 7, 8)).astype(np.float32)))
    W = LO.bf(torch.from_numpy(rng.standard_normal((4, 18 * 8)).astype(np.float32))).numpy()
    b = rng.standard_normal(4).astype(np.float32)
    got = LO.conv233(x, W, b).numpy()
    want = _loop_conv233(x.numpy().astype(np.float64), W, b)
    assert np.abs(got - want).max() <= 2 * 2 ** -7 * np.abs(want).max()


def test_conv233_is_causal():
    rng = np.random.default_rng(1)
    x = LO.bf(torch.from_numpy(rng.standard_normal((1, 2, 4, 4, 8)).astype(np.float32)))
    W = rng.standard_normal((4, 18 * 8)).astype(np.float32)
    b = np.zeros(4, np.float32)
    a = LO.conv233(x, W, b)
    x2 = x.clone()
    x2[:, 1] += 1.0
    assert torch.equal(a[:, 0], LO.conv233(x2, W, b)[:, 0])


def test_fsq_known_answers():
    z = torch.zeros((1, 12))
    codes, idx = LO.fsq(z)
    assert (codes == 0).all()
    # digit = (q + L//2) * basis with q = 0: 4,4,4,2,2,2 over (1,8,64,512,2560,12800)
    assert idx.tolist() == [[32036, 32036]]
    big = LO.fsq(torch.full((1, 12), 50.0))
    assert big[0].tolist()[0] == [0.75, 0.75, 0.75, 1.0, 1.0, 1.0] * 2
    assert big[1].tolist() == [[63999, 63999]]
    small = LO.fsq(torch.full((1, 12), -50.0))
    assert small[0].tolist()[0] == [-1.0] * 12 and small[1].tolist() == [[0, 0]]


def test_fsq_levels_cover_the_codebook():
    z = torch.linspace(-6, 6, 20001)[:, None].repeat(1, 12)
    codes, _ = LO.fsq(z)
    for i, L in enumerate(LO.FSQ_LEVELS):
        assert len(torch.unique(codes[:, i])) == L


def test_dec_in_is_idempotent_on_codes_and_conceals():
    rng = np.random.default_rng(2)
    lv = np.array(LO.FSQ_LEVELS)
    q = rng.integers(-(lv // 2), lv - lv // 2, size=(1, 2, 3, 4, 12))
    codes = q / (lv // 2)
    mask = np.ones((1, 2, 3, 4), np.uint8)
    mask[0, 1, 1, 2] = 0
    mask[0, 0, 2, 3] = 0
    mask[0, 1, 2, 3] = 0
    tok = codes * mask[..., None]
    x = LO.dec_in(tok, mask).numpy()
    assert np.array_equal(x[0, 0, 0, 0, :12], codes[0, 0, 0, 0])
    assert np.array_equal(x[0, 1, 1, 2, :12], codes[0, 0, 1, 2])   # concealed from I
    assert (x[0, 1, 2, 3] == 0).all() and (x[0, 0, 2, 3] == 0).all()  # both lost -> zeros
    assert (x[..., 12:] == 0).all()


def test_weights_are_seeded_bf16_values():
    cfg = LearnedConfig(dim=128, blocks=1, seed=5)
    a, b = make_weights(cfg), make_weights(cfg)
    assert a["W"].keys() == b["W"].keys()
    for k in a["W"]:
        assert np.array_equal(a["W"][k], b["W"][k])
        v = torch.from_numpy(a["W"][k])
        assert torch.equal(v, LO.bf(v))
    assert a["W"]["head"][12:].sum() == 0
    assert a["W"]["dec_in"].reshape(128, 18, 64)[:, :, 12:].sum() == 0
    assert tuple(PROD_LEVELS) == tuple(LO.FSQ_LEVELS)
    with pytest.raises(ValueError):
        LearnedConfig(dim=100)


def test_oracle_end_to_end_small():
    cfg = LearnedConfig(dim=128, blocks=1, seed=0)
    w = make_weights(cfg)
    rng = np.random.default_rng(3)
    fr = rng.random((1, 9, 20, 28, 3), dtype=np.float32)
    codes, idx, hw, _ = LO.encode(fr, 2, w, cfg.blocks)
    assert hw == (10, 14) and codes.shape == (1, 2, 2, 2, 12)
    out = LO.decode(codes, np.ones(codes.shape[:-1], np.uint8), hw, w, cfg.blocks)
    assert out.shape == (1, 9, 10, 14, 3) and out.min() >= 0 and out.max() <= 1


def test_window_attention_matches_bruteforce():
    """The oracle's batched window attention vs a per-query loop (causal in
    latent time, keys restricted to the query's 8x8 window)."""
    rng = np.random.default_rng(9)
    G, T, H, W, D = 1, 2, 10, 11, 128
    qkv = LO.bf(torch.from_numpy(rng.standard_normal((G, T, H, W, 3 * D)).astype(np.float32)))
    got = LO.window_attention(qkv).numpy()
    x = qkv.numpy().astype(np.float64)
    for t in range(T):
        for y in range(H):
            for xx in range(W):
                for hd in range(D // 64):
                    q = x[0, t, y, xx, hd * 64:(hd + 1) * 64] * 0.125
                    keys, vals = [], []
                    for tk in range(t + 1):
                        for yk in range((y // 8) * 8, min(H, (y // 8) * 8 + 8)):
                            for xk in range((xx // 8) * 8, min(W, (xx // 8) * 8 + 8)):
                                keys.append(x[0, tk, yk, xk, D + hd * 64:D + (hd + 1) * 64])
                                vals.append(x[0, tk, yk, xk, 2 * D + hd * 64:2 * D + (hd + 1) * 64])
                    sc = np.array(keys) @ q
                    p = np.exp(sc - sc.max())
                    o = (p / p.sum()) @ np.array(vals)
                    # bf16 output and bf16-rounded probabilities (the P.V operand)
                    np.testing.assert_allclose(got[0, t, y, xx, hd * 64:(hd + 1) * 64], o,
                                               rtol=2 ** -7, atol=4e-3)
