"""GPU: the reference suite's hot-path tests (pkg/tests/test_codec.py,
test_selection.py, test_transport.py token half) run against this package's
drop-in API, plus bit-exact parity against the oracle on seeded inputs of
awkward shapes (odd sizes exercise the non-TMA encoder and edge clamping)."""

import zlib

import numpy as np
import pytest

from helpers import random_gop
from oracle import semstream_oracle as O
from paper_2602_03529_b200 import codec as C, selection as S, transport as T, video as V

pytestmark = pytest.mark.gpu

CFG = C.CodecConfig()


def _gop(frames, gop_id=0):
    return V.GoP(gop_id, tuple(V.Frame(f, timestamp_index=t) for t, f in enumerate(frames)))


def _const_gop(value=0.5, h=16, w=16, gop_id=0):
    return _gop(np.full((9, h, w, 3), value, np.float32), gop_id)


def _bits(a, b):
    return np.array_equal(a, b) and np.array_equal(np.signbit(a), np.signbit(b))


# ---------------------------------------------------------------------------
# test_codec.py

def test_constant_gray_dc_coefficient():
    i, p = C.encode_gop(_const_gop(0.5), CFG)
    assert np.allclose(i.values[:, :, 0::4], 4.0, atol=1e-9)
    assert np.abs(np.delete(i.values, np.s_[0::4], axis=2)).max() < 1e-9
    assert np.allclose(p.values[:, :, 0::4], 4.0, atol=1e-9)


def test_token_shape_contract():
    i, p = C.encode_gop(_const_gop(0.5, 64, 64), CFG)
    assert i.values.shape == (8, 8, 12) and p.values.shape == (8, 8, 12)


def test_encode_determinism(rng):
    g = _gop(random_gop(rng, 24, 24))
    a, b = C.encode_gop(g, CFG), C.encode_gop(g, CFG)
    assert np.array_equal(a[0].values, b[0].values) and np.array_equal(a[1].values, b[1].values)


def test_identical_p_frames_give_identical_p_tokens(rng):
    shared = random_gop(rng)[1:]
    ga = _gop(np.concatenate([random_gop(rng)[:1], shared]))
    gb = _gop(np.concatenate([random_gop(rng)[:1], shared]), 1)
    assert np.array_equal(C.encode_gop(ga, CFG)[1].values, C.encode_gop(gb, CFG)[1].values)


def test_decode_constant_gray_exact():
    g = _const_gop(0.5)
    assert V.gop_psnr(g, C.decode_gop(*C.encode_gop(g, CFG), CFG))[0] == 99.0


def test_decode_conceals_and_partial(rng):
    g = _gop(random_gop(rng))
    i, p = C.encode_gop(g, CFG)
    rec = C.decode_gop(i, C.apply_token_mask(p, np.ones((2, 2), bool)), CFG)
    for t in range(1, 9):
        assert np.array_equal(rec.frames[t].samples, rec.frames[0].samples)
    drop = np.zeros((2, 2), bool)
    drop[0, 0] = True
    part = C.decode_gop(i, C.apply_token_mask(p, drop), CFG)
    full = C.decode_gop(i, p, CFG)
    assert np.array_equal(part.frames[1].samples[:8, :8], part.frames[0].samples[:8, :8])
    assert np.array_equal(part.frames[1].samples[8:, 8:], full.frames[1].samples[8:, 8:])
    again = C.decode_gop(i, C.apply_token_mask(p, np.zeros((2, 2), bool)), CFG)
    for a, b in zip(full.frames, again.frames):
        assert np.array_equal(a.samples, b.samples)
    # frames 1..8 share one buffer, like the reference
    assert full.frames[1].samples is full.frames[8].samples


def test_decode_outputs_in_range(rng):
    for _ in range(5):
        rec = C.decode_gop(*C.encode_gop(_gop(random_gop(rng)), CFG), CFG)
        for f in rec.frames:
            assert f.samples.min() >= 0.0 and f.samples.max() <= 1.0


def test_scaling_kats():
    f = V.Frame(np.full((12, 12, 3), 0.7, np.float32))
    for s in (2, 3):
        d = C.downscale_frame(f, s)
        assert np.allclose(d.samples, 0.7, atol=1e-6)
        assert np.allclose(C.upscale_frame(d, s).samples, 0.7, atol=1e-6)
    arr = np.zeros((2, 2, 3), np.float32)
    arr[0, 1] = 1.0
    arr[1, 1] = 1.0
    d = C.downscale_frame(V.Frame(arr), 2)
    assert d.samples.shape == (1, 1, 3) and np.allclose(d.samples, 0.5)
    e = np.zeros((5, 5, 3), np.float32)
    e[:, 4] = 1.0
    d = C.downscale_frame(V.Frame(e), 3)
    assert d.samples.shape == (2, 2, 3) and d.samples[0, 1, 0] > 0.5


def test_bilinear_matches_oracle(rng):
    img = rng.random((6, 5, 3))
    for s in (2, 3):
        assert _bits(C.bilinear_upscale(img, s), O.bilinear(img, s))


def test_pluggable_upscaler():
    f = V.Frame(np.full((4, 4, 3), 0.25, np.float32))
    up = C.upscale_frame(f, 2, upscaler=lambda img, s: np.repeat(np.repeat(img, s, 0), s, 1))
    assert up.samples.shape == (8, 8, 3) and np.allclose(up.samples, 0.25)


def test_blend_kats(rng):
    zeros, ones = _const_gop(0.0), _const_gop(1.0, gop_id=1)
    b = C.blend_boundary(zeros, ones, 2)
    assert np.allclose(b.frames[0].samples, 0.5) and np.allclose(b.frames[1].samples, 1.0)
    assert np.allclose(b.frames[2].samples, 1.0)
    for _ in range(10):
        prev, curr = _gop(random_gop(rng)), _gop(random_gop(rng), 1)
        before = V.boundary_flicker(prev, curr, 2)
        assert V.boundary_flicker(prev, C.blend_boundary(prev, curr, 2), 2) < before


@pytest.mark.parametrize("n", range(1, 9))
def test_blend_all_widths_match_oracle(rng, n):
    # codec.py:41-42 allows n in 1..8; n >= 5 blends with frames of the
    # previous GoP that were themselves blended
    prev, curr = random_gop(rng, 20, 28), random_gop(rng, 20, 28)
    out = C.blend_boundary(_gop(prev), _gop(curr, 1), n)
    want = O.blend(list(prev), list(curr), n)
    for a, b in zip(out.frames, want):
        assert _bits(a.samples, b)


def test_scale_gop_roundtrip_shapes(rng):
    g = _gop(random_gop(rng, 30, 30))
    down = C.scale_gop(g, 3, "down")
    assert (down.height, down.width, down.scale) == (10, 10, 3)
    up = C.scale_gop(down, 3, "up", crop=(30, 30))
    assert (up.height, up.width) == (30, 30)


# ---------------------------------------------------------------------------
# test_selection.py

def _tok(kind, v):
    v = np.asarray(v, np.float64)
    return C.TokenMatrix(kind, v, np.ones(v.shape[:2], bool))


def test_similarity_kats():
    v = np.arange(1, 13, dtype=np.float64).reshape(1, 1, 12)
    assert S.token_similarity(_tok("P", v), _tok("I", v.copy())).values[0, 0] == pytest.approx(1.0)
    p, i = np.zeros((1, 2, 12)), np.zeros((1, 2, 12))
    i[0, 1, 0] = 2.0
    s = S.token_similarity(_tok("P", p), _tok("I", i)).values
    assert s[0, 0] == 1.0 and s[0, 1] == 0.0
    p, i = np.zeros((1, 1, 12)), np.zeros((1, 1, 12))
    p[0, 0, :2] = [1.0, 1.0]
    i[0, 0, :2] = [1.0, 0.0]
    assert S.token_similarity(_tok("P", p), _tok("I", i)).values[0, 0] == \
        pytest.approx(0.7071067811865476, abs=1e-6)


def test_similarity_scale_invariance_and_parity(rng):
    p = rng.random((4, 4, 12)) - 0.2
    i = rng.random((4, 4, 12)) - 0.2
    a = S.token_similarity(_tok("P", p), _tok("I", i)).values
    b = S.token_similarity(_tok("P", 37.5 * p), _tok("I", 0.004 * i)).values
    assert np.abs(a - b).max() < 1e-12
    assert _bits(a, O.similarity(p, i))
    for c in (1, 3, 7, 8, 13, 16, 40):           # other widths: numpy pairwise order
        p, i = rng.standard_normal((5, 6, c)), rng.standard_normal((5, 6, c))
        got = S.token_similarity(_tok("P", p), _tok("I", i)).values
        assert _bits(got, O.similarity(p, i)), c


def test_drop_masks(rng):
    sim = S.SimilarityMap(rng.uniform(-1, 1, (8, 8)))
    assert not S.build_drop_mask(sim, 0.0).any()
    m = S.build_drop_mask(sim, 0.25)
    assert int(m.sum()) == 16 and sim.values[m].min() >= sim.values[~m].max() - 1e-12
    for _ in range(10):
        values = rng.uniform(-1, 1, (6, 7))
        k = int(rng.integers(0, values.size + 1))
        mask = S.top_k_drop_mask(S.SimilarityMap(values), k)
        pairs = sorted(((-v, idx) for idx, v in enumerate(values.ravel())))
        assert set(np.flatnonzero(mask.ravel())) == {idx for _, idx in pairs[:k]}
    assert np.array_equal(S.top_k_drop_mask(S.SimilarityMap(np.full((2, 3), 0.5)), 4).ravel(),
                          [1, 1, 1, 1, 0, 0])
    prev = np.zeros((8, 8), bool)
    for rate in (0.05, 0.10, 0.15, 0.20, 0.25, 0.30):
        cur = S.build_drop_mask(sim, rate)
        assert (prev <= cur).all()
        prev = cur


def test_topk_massive_ties_large(rng):
    # static content: most similarities exactly 1.0 -- the tie-break decides
    vals = np.where(rng.random((68, 120)) < 0.77, 1.0, rng.choice([0.5, 0.25, -0.0, 0.0], (68, 120)))
    sim = S.SimilarityMap(vals)
    for k in (0, 1, 816, 2448, 6283, 8159, 8160):
        assert np.array_equal(S.top_k_drop_mask(sim, k), O.top_k_mask(vals, k)), k


def test_similarity_beats_random_on_moving_square():
    from oracle.synth import make_clip
    g = _gop(make_clip("moving-square", 64, 64, 9, seed=5).gop(0))
    i, p = C.encode_gop(g, CFG)
    sim = S.token_similarity(p, i)
    k = sim.values.size // 2
    _, mse_sim = V.gop_psnr(g, C.decode_gop(i, C.apply_token_mask(p, S.top_k_drop_mask(sim, k)), CFG))
    wins = 0
    for s in range(20):
        r = np.random.default_rng(s)
        flat = np.zeros(sim.values.size, bool)
        flat[r.choice(sim.values.size, size=k, replace=False)] = True
        rec = C.decode_gop(i, C.apply_token_mask(p, flat.reshape(sim.values.shape)), CFG)
        wins += mse_sim < V.gop_psnr(g, rec)[1]
    assert wins >= 19


# ---------------------------------------------------------------------------
# test_transport.py (token packets)

def _matrix(rng, h=8, w=8, c=12, kind="P", gop_id=0, mask=None):
    values = rng.uniform(-4.0, 4.0, (h, w, c))
    if mask is None:
        mask = np.ones((h, w), bool)
    return C.TokenMatrix(kind, np.where(mask[..., None], values, 0.0), mask, gop_id=gop_id)


def test_packet_counts_sizes_and_bytes(rng):
    m = _matrix(rng)
    pk = T.packetize_tokens(m, scale=2)
    assert len(pk) == 8
    for p in pk:
        assert p.mask.all() and len(p.payload) == 96
        assert len(p.to_bytes()) == T.token_packet_wire_size(8, 12)
    assert [p.to_bytes() for p in pk] == O.packetize(O.KIND_P, 0, m.values, m.mask, 2)


def test_header_only_and_constant_rows(rng):
    mask = np.ones((8, 8), bool)
    mask[3] = False
    pk = T.packetize_tokens(_matrix(rng, mask=mask))
    assert pk[3].payload == b"" and not pk[3].mask.any() and pk[3].quant_range == 0.0
    m = C.TokenMatrix("I", np.full((2, 8, 12), 1.234), np.ones((2, 8), bool))
    pk = T.packetize_tokens(m)
    assert pk[0].quant_range == 0.0 and pk[0].payload == bytes(96)
    back = T.reassemble(pk, (2, 8, 12), "I")
    assert np.abs(back.values - np.float32(1.234)).max() < 1e-6


def test_wire_roundtrip_quantizer_bound(rng):
    m = _matrix(rng)
    pk = T.parse_packets([p.to_bytes() for p in T.packetize_tokens(m)])
    back = T.reassemble(pk, (8, 8, 12), "P")
    for r in range(8):
        qr = max(float(m.values[r].max() - m.values[r].min()), 0.0)
        assert np.abs(back.values[r] - m.values[r]).max() <= qr / 510 + 1e-5
    assert np.array_equal(back.mask, m.mask)


def test_byte_stability_and_prefix(rng):
    m = _matrix(rng, h=2, w=3, c=2)
    a = [p.to_bytes() for p in T.packetize_tokens(m, scale=3)]
    assert a == [p.to_bytes() for p in T.packetize_tokens(m, scale=3)]
    assert a[0][:4] == bytes([0x4D, 0x53, 0x01, 0x01])


def test_crc_flip_and_errors(rng):
    data = bytearray(T.packetize_tokens(_matrix(rng, h=1, w=4, c=2))[0].to_bytes())
    data[10] ^= 0xFF
    with pytest.raises(T.PacketFormatError, match="crc"):
        T.parse_packet(bytes(data))
    with pytest.raises(T.PacketFormatError, match="shorter"):
        T.parse_packet(b"\x00\x01")
    body = b"\x00\x00\x01\x00" + bytes(20)
    with pytest.raises(T.PacketFormatError, match="magic"):
        T.parse_packet(body + zlib.crc32(body).to_bytes(4, "big"))
    body = b"\x4d\x53\x02\x00" + bytes(20)
    with pytest.raises(T.PacketFormatError, match="version"):
        T.parse_packet(body + zlib.crc32(body).to_bytes(4, "big"))
    good = T.packetize_tokens(_matrix(rng, h=1, w=4, c=2))[0].to_bytes()
    body = good[:-5]                                   # drop one payload byte
    with pytest.raises(T.PacketFormatError, match="payload length"):
        T.parse_packet(body + zlib.crc32(body).to_bytes(4, "big"))


def test_reassembly_rules(rng):
    assert not T.reassemble([], (4, 4, 12), "I").mask.any()
    m = _matrix(rng, h=2, w=4, c=3)
    first = T.packetize_tokens(m)
    other = T.packetize_tokens(_matrix(rng, h=2, w=4, c=3))
    out = T.reassemble([first[0], other[0], first[1]], (2, 4, 3), "P")
    assert np.array_equal(out.values, T.reassemble(first, (2, 4, 3), "P").values)
    rogue = T.TokenPacket(kind="P", gop_id=0, row_index=7, width_tokens=4, channels=3, scale=1,
                          quant_min=0.0, quant_range=0.0, mask=np.zeros(4, bool), payload=b"")
    stats = {}
    out = T.reassemble(T.packetize_tokens(m) + [rogue], (2, 4, 3), "P", stats=stats)
    assert stats["corrupt"] == 1 and stats["rows_received"] == 2 and out.mask.all()
    # caller-built packets whose payload does not hold popcount(mask)*C bytes:
    # the reference's dequantized() reshape raises; a row that is never
    # dequantised (duplicate) is ignored, as in the reference
    good = first[0]
    for pay in (good.payload[:-1], good.payload + b"\0"):
        bad = T.TokenPacket(kind="P", gop_id=0, row_index=0, width_tokens=4, channels=3, scale=1,
                            quant_min=good.quant_min, quant_range=good.quant_range,
                            mask=good.mask, payload=pay)
        with pytest.raises(ValueError):
            T.reassemble([bad], (2, 4, 3), "P")
        out = T.reassemble([good, bad, first[1]], (2, 4, 3), "P")
        assert np.array_equal(out.values, T.reassemble(first, (2, 4, 3), "P").values)


def test_sender_drop_equals_network_loss(rng):
    for _ in range(10):
        h, w, c = 6, 5, 4
        mask = rng.random((h, w)) > 0.3
        lost = set(int(r) for r in rng.choice(h, size=2, replace=False))
        values = rng.uniform(-1, 1, (h, w, c))
        ma = C.TokenMatrix("P", np.where(mask[..., None], values, 0.0), mask)
        out_a = T.reassemble([p for p in T.packetize_tokens(ma) if p.row_index not in lost],
                             (h, w, c), "P")
        mb = mask.copy()
        for r in lost:
            mb[r] = False
        out_b = T.reassemble(T.packetize_tokens(C.TokenMatrix("P", np.where(mb[..., None], values, 0.0), mb)),
                             (h, w, c), "P")
        assert out_a.values.tobytes() == out_b.values.tobytes()
        assert np.array_equal(out_a.mask, out_b.mask)


def test_golden_wire_bytes():
    mask = np.array([True, False, True])
    pkt = T.TokenPacket(kind="I", gop_id=0x01020304, row_index=5, width_tokens=3, channels=1,
                        scale=2, quant_min=0.0, quant_range=1.0, mask=mask, payload=b"\x00\xff")
    data = pkt.to_bytes()
    body = (b"\x4d\x53\x01\x00\x01\x02\x03\x04\x00\x05\x00\x03\x01\x02"
            b"\x00\x00\x00\x00\x3f\x80\x00\x00\xa0\x00\xff")
    assert data[:-4] == body and data[-4:] == zlib.crc32(body).to_bytes(4, "big")
    back = T.parse_packet(data)
    assert back.row_index == 5 and back.scale == 2 and np.array_equal(back.mask, mask)
    assert np.array_equal(back.dequantized(), [[0.0], [1.0]])


# ---------------------------------------------------------------------------
# parity vs the oracle on awkward shapes

@pytest.mark.parametrize("hw", [(5, 7), (16, 16), (30, 30), (37, 61), (62, 102), (170, 250),
                                (72, 96)])
def test_api_parity_awkward_shapes(rng, hw):
    h, w = hw
    frames = rng.random((9, h, w, 3)).astype(np.float32)
    g = _gop(frames)
    for s in (2, 3):
        work = C.scale_gop(g, s, "down")
        assert _bits(work.stacked(), O.downscale(frames, s))
        i, p = C.encode_gop(work, CFG)
        oi, op = O.encode(O.downscale(frames, s))
        assert _bits(i.values, oi) and _bits(p.values, op)
        rec = C.decode_gop(i, p, CFG)
        ri, rp = O.decode(oi, op, np.ones(oi.shape[:2], bool), work.stacked().shape[1:3])
        assert _bits(rec.frames[0].samples, ri) and _bits(rec.frames[1].samples, rp)
        up = C.scale_gop(rec, s, "up", crop=(h, w))
        assert _bits(up.frames[0].samples, O.upscale(ri, s, (h, w)))
    i, p = C.encode_gop(g, CFG)                      # direct (s = 1) tokenizer
    oi, op = O.encode(frames)
    assert _bits(i.values, oi) and _bits(p.values, op)


# ---------------------------------------------------------------------------
# size extremes

def test_large_packets_crc_beyond_shift_table(rng):
    # 3000-token rows: ~36 KB packets, so lane chunks sit > 4096 bytes from the
    # end and the CRC merge takes the square-and-multiply path
    h, w, c = 2, 3000, 12
    vals = rng.uniform(-3, 3, (h, w, c))
    mask = rng.random((h, w)) > 0.2
    vals = np.where(mask[..., None], vals, 0.0)
    m = C.TokenMatrix("P", vals, mask, gop_id=77)
    pk = T.packetize_tokens(m, scale=3)
    wire = [p.to_bytes() for p in pk]
    assert wire == O.packetize(O.KIND_P, 77, vals, mask, 3)
    assert len(wire[0]) > 25000
    back = T.reassemble(T.parse_packets(wire), (h, w, c), "P", gop_id=77)
    ov, om = O.reassemble([O.parse(d) for d in wire], (h, w, c))
    assert _bits(back.values, ov) and np.array_equal(back.mask, om)
    # field-wise serialisation of the same packets (user-built TokenPacket)
    rebuilt = [T.TokenPacket(p.kind, p.gop_id, p.row_index, p.width_tokens, p.channels, p.scale,
                             p.quant_min, p.quant_range, p.mask, p.payload) for p in pk]
    assert [p.to_bytes() for p in rebuilt] == wire


def test_many_rows_and_single_column(rng):
    # tall, 1-token-wide matrices: 20000 row packets in one launch
    h, w, c = 20000, 1, 3
    vals = rng.uniform(-1, 1, (h, w, c))
    m = C.TokenMatrix("I", vals, np.ones((h, w), bool), gop_id=5)
    wire = [p.to_bytes() for p in T.packetize_tokens(m)]
    assert wire == O.packetize(O.KIND_I, 5, vals, np.ones((h, w), bool), 1)


def test_empty_and_all_dropped_rows(rng):
    m = C.TokenMatrix("P", np.zeros((3, 5, 12)), np.zeros((3, 5), bool))
    pk = T.packetize_tokens(m)
    assert all(p.payload == b"" and p.quant_range == 0.0 for p in pk)
    back = T.reassemble(T.parse_packets([p.to_bytes() for p in pk]), (3, 5, 12), "P")
    assert not back.mask.any() and not back.values.any()
    assert T.packetize_tokens(C.TokenMatrix("I", np.zeros((0, 4, 12)), np.zeros((0, 4), bool))) == []
