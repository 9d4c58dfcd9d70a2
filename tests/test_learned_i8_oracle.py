"""CPU: the exact int8 learned-tokenizer oracle (oracle/learned_i8_oracle.py)
checked against brute-force loop restatements on tiny shapes -- integer GEMM,
(2,3,3) causal im2col, requantisation, the integer window attention, FSQ and
the decoder-input gather -- and the model definition's invariants."""

import numpy as np

from oracle import learned_i8_oracle as LO
from paper_2602_03529_b200.learned_i8 import (LearnedI8Config, exp_table, make_weights_i8,
                                              silu_table)


def test_gemm_exact_vs_int64():
    rng = np.random.default_rng(0)
    x = rng.integers(-128, 128, (7, 4608)).astype(np.int8)
    W = rng.integers(-127, 128, (5, 4608)).astype(np.int8)
    want = x.astype(np.int64) @ W.astype(np.int64).T
    assert np.array_equal(LO.gemm(x, W), want)
    x[:] = 127
    W[:] = 127
    assert (LO.gemm(x, W) == 4608 * 127 * 127).all()           # < 2^31: int32 TMEM is exact


def test_im2col_causal_loops():
    rng = np.random.default_rng(1)
    x = rng.integers(-9, 9, (1, 2, 3, 4, 2)).astype(np.int8)
    cols = LO.im2col233(x)
    for t in range(2):
        for y in range(3):
            for xx in range(4):
                for tap, (dt, dy, dx) in enumerate(LO.TAPS_233):
                    tt, yy, xq = t + dt, y + dy, xx + dx
                    want = x[0, tt, yy, xq] if (tt >= 0 and 0 <= yy < 3 and 0 <= xq < 4) else 0
                    assert np.array_equal(cols[0, t, y, xx, tap * 2:(tap + 1) * 2], want * np.ones(2))


def test_requant_rounding_and_saturation():
    acc = np.array([-2048 - 1024, -1024, -1023, 0, 1023, 1024, 10 ** 7, -(10 ** 7)])
    y = LO.requant(acc, np.zeros(8, np.int64), 11)
    assert y.tolist() == [-1, 0, 0, 0, 0, 1, 127, -127]       # floor((x + 1024) / 2048)
    lut = silu_table()
    assert LO.requant(np.array([0]), np.array([0]), 1, lut).tolist() == [0]
    assert LO.requant(np.array([200]), np.array([0]), 1, None, np.array([100])).tolist() == [127]


def test_attention_core_loops():
    rng = np.random.default_rng(2)
    Ht, Wt, D = 3, 10, 256
    qkv = rng.integers(-40, 40, (1, 2, Ht, Wt, 3 * D)).astype(np.int8)
    lut = exp_table()
    got = LO.attention_core(qkv, D, 128, 8, lut)
    for h in range(2):
        for t in range(2):
            for y in range(Ht):
                for x in range(Wt):
                    wy, wx = y // 8, x // 8
                    keys = [(tt, yy, xq) for tt in range(t + 1) for yy in range(wy * 8, min(wy * 8 + 8, Ht))
                            for xq in range(wx * 8, min(wx * 8 + 8, Wt))]
                    q = qkv[0, t, y, x, h * 128:(h + 1) * 128].astype(np.int64)
                    S = [int(q @ qkv[0, tt, yy, xq, D + h * 128:D + (h + 1) * 128].astype(np.int64))
                         for tt, yy, xq in keys]
                    m = max(S)
                    e = [int(lut[min((m - s) >> 8, 255)]) for s in S]
                    l_ = sum(e)
                    for d in (0, 77, 127):
                        O = sum(ei * int(qkv[0, tt, yy, xq, 2 * D + h * 128 + d])
                                for ei, (tt, yy, xq) in zip(e, keys))
                        want = max(-127, min(127, (2 * O + l_) // (2 * l_)))
                        assert got[0, t, y, x, h * 128 + d] == want


def test_fsq_levels_and_indices():
    acc = np.zeros((1, 16), np.int64)
    acc[0, :12] = np.array([-99, 99, 0, -99, 99, 0, 1, 2, 3, 4, 5, 6]) << 13
    codes, idx = LO.fsq(acc, np.zeros(16, np.int64), 13)
    assert codes[0, :6].tolist() == [-1.0, 0.75, 0.0, -1.0, 1.0, 0.0]
    L = np.array(LO.FSQ_LEVELS)
    q = np.rint(codes[0] * (L // 2)).astype(int) + L // 2
    assert idx[0, 0] == sum(int(q[i]) * LO.BASIS[i] for i in range(6))
    assert 0 <= idx.min() and idx.max() < 8 * 8 * 8 * 5 * 5 * 5


def test_dec_input_concealment():
    tok = np.zeros((1, 2, 2, 2, 12))
    tok[0, 0] = 0.5
    mask = np.ones((1, 2, 2, 2), np.uint8)
    mask[0, 1, 0, 0] = 0                                          # dropped P token
    q = LO.snap_codes(tok, mask)
    assert np.array_equal(q[0, 1, 0, 0], q[0, 0, 0, 0]) and (q[0, 1, 1, 1] == 0).all()
    x = LO.dec_input(q)
    assert x.shape == (1, 2, 2, 2, 256) and (x[..., 216:] == 0).all()


def test_model_definition():
    w = make_weights_i8(LearnedI8Config())
    assert all(v.dtype == np.int8 for v in w["W"].values())
    assert all(v.dtype == np.int32 for v in w["b"].values())
    assert (w["W"]["pe_i"][:, 192:] == 0).all() and (w["W"]["dec_in"][:, 216:] == 0).all()
    assert all(1 <= s <= 20 for s in w["sh"].values())
    assert exp_table()[0] == 255 and exp_table()[255] == 0
    assert make_weights_i8(LearnedI8Config())["W"]["enc0_c1"].tobytes() == w["W"]["enc0_c1"].tobytes()


def test_encode_decode_small_deterministic():
    from oracle.synth import make_clip
    w = make_weights_i8(LearnedI8Config())
    clip = make_clip("moving-square", 64, 48, 9, seed=1)
    fr = clip.gop(0)[None]
    c1, i1, hw = LO.encode(fr, 1, w)
    c2, i2, _ = LO.encode(fr, 1, w)
    assert np.array_equal(i1, i2) and hw == (48, 64)
    dec = LO.decode(c1, np.ones(c1.shape[:-1], np.uint8), hw, w)
    assert dec.shape == (1, 9, 48, 64, 3) and dec.min() >= 0 and dec.max() <= 1


def test_haar_front_loops():
    """haar_front against a loop restatement: temporal levels over the eight
    P frames, then spatial levels (rows, then columns) on every frame slot."""
    def step(v):                                    # one level over a list
        m = len(v)
        lo = [(v[2 * j] + v[2 * j + 1]) >> 1 for j in range(m // 2)]
        hi = [(v[2 * j] - v[2 * j + 1]) >> 1 for j in range(m // 2)]
        return lo + hi

    rng = np.random.default_rng(5)
    q = rng.integers(-128, 128, (1, 1, 2, 9, 8, 8, 3))
    got = LO.haar_front(q)
    want = q.astype(np.int64).copy()
    for tx in range(2):
        for y in range(8):
            for x in range(8):
                for c in range(3):
                    v = [int(want[0, 0, tx, 1 + f, y, x, c]) for f in range(8)]
                    for m in (8, 4, 2):
                        v[:m] = step(v[:m])
                    want[0, 0, tx, 1:, y, x, c] = v
        for f in range(9):
            for c in range(3):
                a = want[0, 0, tx, f, :, :, c].tolist()
                for m in (8, 4, 2):
                    for y in range(m):
                        a[y][:m] = step(a[y][:m])
                    for x in range(m):
                        col = step([a[y][x] for y in range(m)])
                        for y in range(m):
                            a[y][x] = col[y]
                want[0, 0, tx, f, :, :, c] = a
    assert np.array_equal(got, want)
    assert got.min() >= -128 and got.max() <= 127
    flat = LO.haar_front(np.full((1, 1, 1, 9, 8, 8, 3), -77))   # flat GoP: DC only
    assert np.count_nonzero(flat) == 6 and (flat[0, 0, 0, :2, 0, 0] == -77).all()
