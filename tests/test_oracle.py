"""CPU: the oracle (oracle/) pinned against the reference's golden vectors,
known-answer tests and the golden fixtures generated from the live reference.
No GPU, no /root/reference needed."""

import math
import struct
import zlib

import numpy as np
import pytest
from scipy.fft import dct, dctn, idct, idctn

from helpers import case_clip, digest, golden, golden_cases, oracle_case, random_gop, wire_digest
from oracle import semstream_oracle as O
from oracle.dct8 import dct2_last, dct3_last, dctn2_8x8, idctn2_8x8


# ---------------------------------------------------------------------------
# ducc0 DCT restatement vs scipy (the reference's third-party dependency)

def _same_bits(a, b):
    return np.array_equal(a, b) and np.array_equal(np.signbit(a), np.signbit(b))


def test_dct_1d_bit_exact_vs_scipy():
    rng = np.random.default_rng(5)
    x = rng.random((20000, 8)) * rng.choice([1.0, 1e-3, 1e3], (20000, 1))
    assert _same_bits(dct2_last(x), dct(x, type=2, norm="ortho"))
    assert _same_bits(dct3_last(x), idct(x, type=2, norm="ortho"))


def test_dctn_bit_exact_vs_scipy():
    rng = np.random.default_rng(6)
    b = rng.standard_normal((8000, 8, 8))
    assert _same_bits(dctn2_8x8(b), dctn(b, type=2, norm="ortho", axes=(-2, -1)))
    assert _same_bits(idctn2_8x8(b), idctn(b, type=2, norm="ortho", axes=(-2, -1)))


def test_idctn_sparse_decoder_inputs_bit_exact():
    rng = np.random.default_rng(7)
    c = np.zeros((6000, 8, 8))
    c[:, 0, 0] = rng.random(6000) * 8
    c[:, 0, 1] = rng.standard_normal(6000)
    c[:, 1, 0] = rng.standard_normal(6000)
    c[:, 2, 0] = rng.standard_normal(6000)
    c[::5, 0, 1] = 0.0
    c[::7] = 0.0
    assert _same_bits(idctn2_8x8(c), idctn(c, type=2, norm="ortho", axes=(-2, -1)))


def test_dct_constant_blocks():
    z = np.zeros((4, 8, 8))
    z[1:] = np.array([0.5, 0.123, 1.0])[:, None, None]
    assert _same_bits(dctn2_8x8(z), dctn(z, type=2, norm="ortho", axes=(-2, -1)))


# ---------------------------------------------------------------------------
# known-answer tests restated from pkg/tests/test_codec.py

def test_constant_gray_dc_coefficient():
    # test_codec.py:39-47: DC = 8 * 0.5 = 4 for the orthonormal 8x8 DCT-II
    gop = np.full((9, 16, 16, 3), 0.5, np.float32)
    i_vals, p_vals = O.encode(gop)
    assert np.allclose(i_vals[:, :, 0::4], 4.0, atol=1e-9)
    assert np.abs(np.delete(i_vals, np.s_[0::4], axis=2)).max() < 1e-9
    assert np.allclose(p_vals[:, :, 0::4], 4.0, atol=1e-9)


def test_token_shape_contract():
    # test_codec.py:50-56
    i_vals, _ = O.encode(np.full((9, 64, 64, 3), 0.5, np.float32))
    assert i_vals.shape == (8, 8, 12)
    assert O.token_grid_shape(60, 50) == (8, 7)


def test_downscale_kats():
    # test_codec.py:186-213
    arr = np.zeros((2, 2, 3), np.float32)
    arr[0, 1] = 1.0
    arr[1, 1] = 1.0
    assert np.allclose(O.downscale(arr, 2), 0.5)
    yy, xx = np.meshgrid(np.arange(64), np.arange(64), indexing="ij")
    checker = np.repeat(((yy + xx) % 2).astype(np.float32)[:, :, None], 3, axis=2)
    assert np.allclose(O.downscale(checker, 2), 0.5, atol=1e-6)
    edge = np.zeros((5, 5, 3), np.float32)
    edge[:, 4] = 1.0
    d = O.downscale(edge, 3)
    assert d.shape == (2, 2, 3) and d[0, 1, 0] > 0.5


def _bilinear_loop(img, s):
    # per-pixel loop oracle of test_codec.py:231-245
    h, w = img.shape[:2]
    out = np.zeros((h * s, w * s, 3))
    for oy in range(h * s):
        for ox in range(w * s):
            sy = min(max((oy + 0.5) / s - 0.5, 0.0), h - 1.0)
            sx = min(max((ox + 0.5) / s - 0.5, 0.0), w - 1.0)
            y0, x0 = int(math.floor(sy)), int(math.floor(sx))
            y1, x1 = min(y0 + 1, h - 1), min(x0 + 1, w - 1)
            fy, fx = sy - y0, sx - x0
            for c in range(3):
                top = img[y0, x0, c] * (1 - fx) + img[y0, x1, c] * fx
                bot = img[y1, x0, c] * (1 - fx) + img[y1, x1, c] * fx
                out[oy, ox, c] = top * (1 - fy) + bot * fy
    return out


def test_bilinear_matches_loop_oracle(rng):
    img = rng.random((6, 5, 3))
    for s in (2, 3):
        assert np.array_equal(O.bilinear(img, s), _bilinear_loop(img, s))


def test_decode_matches_truncation(rng):
    # test_codec.py:84-110 truncation oracle with explicit basis matrices
    n = 8
    m = np.array([[(math.sqrt(1 / n) if k == 0 else math.sqrt(2 / n)) *
                   math.cos(math.pi * (2 * i + 1) * k / (2 * n)) for i in range(n)]
                  for k in range(n)])
    gop = random_gop(rng, dyadic=True)
    i_vals, p_vals = O.encode(gop)
    i_img, _ = O.decode(i_vals, p_vals, np.ones(i_vals.shape[:2], bool), (16, 16))
    src = gop[0].astype(np.float64)
    expect = np.empty_like(src)
    for by in range(2):
        for bx in range(2):
            for c in range(3):
                blk = src[by * 8:(by + 1) * 8, bx * 8:(bx + 1) * 8, c]
                co = m @ blk @ m.T
                kept = np.zeros_like(co)
                for (y, x) in O.COEFF_POSITIONS:
                    kept[y, x] = co[y, x]
                expect[by * 8:(by + 1) * 8, bx * 8:(bx + 1) * 8, c] = m.T @ kept @ m
    assert np.abs(i_img - np.clip(expect, 0, 1)).max() < 1e-6


def test_similarity_kats():
    # test_selection.py:18-49
    v = np.arange(1, 13, dtype=np.float64).reshape(1, 1, 12)
    assert O.similarity(v, v.copy())[0, 0] == pytest.approx(1.0)
    p = np.zeros((1, 1, 12))
    i = np.zeros((1, 1, 12))
    p[0, 0, 0] = 1.0
    i[0, 0, 1] = 1.0
    assert O.similarity(p, i)[0, 0] == pytest.approx(0.0)
    p = np.zeros((1, 1, 12))
    i = np.zeros((1, 1, 12))
    p[0, 0, :2] = [1.0, 1.0]
    i[0, 0, :2] = [1.0, 0.0]
    assert O.similarity(p, i)[0, 0] == pytest.approx(0.7071067811865476, abs=1e-6)
    p = np.zeros((1, 2, 12))
    i = np.zeros((1, 2, 12))
    i[0, 1, 0] = 2.0
    s = O.similarity(p, i)
    assert s[0, 0] == 1.0 and s[0, 1] == 0.0


def test_top_k_tie_break_row_major():
    # test_selection.py:98-101
    mask = O.top_k_mask(np.full((2, 3), 0.5), 4)
    assert np.array_equal(mask.ravel(), [1, 1, 1, 1, 0, 0])


def test_top_k_full_sort_oracle(rng):
    # test_selection.py:86-95
    for _ in range(10):
        values = rng.uniform(-1, 1, (6, 7))
        k = int(rng.integers(0, values.size + 1))
        mask = O.top_k_mask(values, k)
        pairs = sorted(((-v, idx) for idx, v in enumerate(values.ravel())))
        assert set(np.flatnonzero(mask.ravel())) == {idx for _, idx in pairs[:k]}


def test_reference_golden_wire_bytes():
    # pkg/tests/test_transport.py:164-189: the only frozen golden packet of the
    # reference suite.  Restated through the oracle's parser and zlib.
    body = (b"\x4d\x53" b"\x01" b"\x00" b"\x01\x02\x03\x04" b"\x00\x05" b"\x00\x03" b"\x01"
            b"\x02" b"\x00\x00\x00\x00" b"\x3f\x80\x00\x00" b"\xa0" b"\x00\xff")
    data = body + zlib.crc32(body).to_bytes(4, "big")
    pk = O.parse(data)
    assert pk["row"] == 5 and pk["scale"] == 2 and pk["gop_id"] == 0x01020304
    assert np.array_equal(pk["mask"], [True, False, True])
    assert pk["payload"] == b"\x00\xff"
    bad = bytearray(data)
    bad[10] ^= 0xFF
    with pytest.raises(O.OraclePacketError, match="crc"):
        O.parse(bytes(bad))


def test_quantiser_bound_and_roundtrip(rng):
    # test_transport.py:52-60: |err| <= qrange/510 + 1e-5
    vals = rng.uniform(-4, 4, (8, 8, 12))
    mask = np.ones((8, 8), bool)
    wire = O.packetize(O.KIND_P, 0, vals, mask)
    back, bm = O.reassemble([O.parse(d) for d in wire], (8, 8, 12))
    for r in range(8):
        qr = float(vals[r].max() - vals[r].min())
        assert np.abs(back[r] - vals[r]).max() <= qr / 510 + 1e-5
    assert bm.all()
    assert len(wire[0]) == O.wire_size(8, 12)


# ---------------------------------------------------------------------------
# golden fixtures generated from the live reference (tests/golden/make_golden.py)

def test_golden_file_provenance():
    g = golden()
    assert "make_golden.py" in g["generator"]
    assert len(g["cases"]) >= 6


@pytest.mark.parametrize("c", golden_cases(max_pixels=1280 * 720),
                         ids=[c["case"]["name"] for c in golden_cases(max_pixels=1280 * 720)])
def test_oracle_matches_reference_golden(c):
    for rec, frames, res in oracle_case(c):
        assert digest(frames) == rec["src"], "synth port differs from the reference clip"
        assert digest(res["work"]) == rec["work"]
        assert digest(res["i_vals"]) == rec["tok_i"]
        assert digest(res["sim"]) == rec["sim"]
        assert digest(res["drop"].astype(np.uint8)) == rec["drop"]
        assert digest(res["p_vals"]) == rec["tok_p"]
        assert wire_digest(res["wire"]) == rec["wire"]
        assert list(res["rows_received"]) == rec["rows_received"]
        assert digest(res["i_img"]) == rec["i_img"]
        assert digest(res["p_img"]) == rec["p_img"]
        assert digest(np.stack(res["frames"])) == rec["out"]
        if rec["wire_first"]:
            assert res["wire"][0].hex() == rec["wire_first"]


@pytest.mark.slow
def test_oracle_matches_reference_golden_1080p():
    c = [c for c in golden_cases() if c["case"]["name"].startswith("c3_")][0]
    for rec, frames, res in oracle_case(c):
        assert digest(res["i_vals"]) == rec["tok_i"]
        assert digest(res["drop"].astype(np.uint8)) == rec["drop"]
        assert wire_digest(res["wire"]) == rec["wire"]
        assert digest(np.stack(res["frames"])) == rec["out"]
