"""CPU: host-side logic of the drop-in API -- validation, error types and
messages that the reference suite pins, geometry -- none of which touches the
GPU; plus "no CPU fallback": product calls fail loudly without CUDA."""

import numpy as np
import pytest
import torch

import paper_2602_03529_b200 as P
from paper_2602_03529_b200 import codec as C, selection as S, transport as T, video as V


def test_codec_config_validation():
    # codec.py:36-46
    C.CodecConfig()
    with pytest.raises(ValueError):
        C.CodecConfig(spatial_factor=4)
    with pytest.raises(ValueError):
        C.CodecConfig(scale=4)
    with pytest.raises(ValueError):
        C.CodecConfig(blend_width=9)
    with pytest.raises(ValueError):
        C.CodecConfig(channels=10)


def test_token_matrix_invariants():
    # codec.py:63-79; test_codec.py:196-200
    with pytest.raises(ValueError):
        C.TokenMatrix("P", np.ones((2, 2, 12)), np.zeros((2, 2), bool))
    with pytest.raises(ValueError):
        C.TokenMatrix("X", np.zeros((2, 2, 12)), np.zeros((2, 2), bool))
    with pytest.raises(ValueError):
        C.TokenMatrix("I", np.zeros((2, 2)), np.zeros((2, 2), bool))
    with pytest.raises(ValueError):
        C.TokenMatrix("I", np.full((1, 1, 12), np.nan), np.ones((1, 1), bool))
    m = C.TokenMatrix("I", np.zeros((3, 4, 12)), np.ones((3, 4), bool), frame_shape=[20, 30])
    assert (m.height_tokens, m.width_tokens, m.channels) == (3, 4, 12)
    assert m.frame_shape == (20, 30)


def test_frame_and_gop_validation():
    with pytest.raises(ValueError):
        V.Frame(np.zeros((4, 4)))
    with pytest.raises(ValueError):
        V.Frame(np.full((4, 4, 3), 1.5, np.float32))
    with pytest.raises(ValueError):
        V.Frame(np.full((4, 4, 3), np.inf, np.float32))
    f = V.Frame(np.zeros((4, 5, 3), np.float32))
    with pytest.raises(ValueError):
        V.GoP(0, (f,) * 8)
    with pytest.raises(ValueError):
        V.GoP(0, (f,) * 8 + (V.Frame(np.zeros((5, 5, 3), np.float32)),))
    with pytest.raises(ValueError):
        V.GoP(0, (f,) * 9, scale=4)


def test_segment_gops_tail_padding():
    # video.py:236-251
    frames = [V.Frame(np.full((2, 2, 3), i / 20, np.float32), i) for i in range(20)]
    gops = V.segment_gops(frames, start_gop_id=5)
    assert [g.gop_id for g in gops] == [5, 6, 7]
    assert gops[-1].frames[-1] is frames[-1] and gops[-1].frames[2] is frames[-1]
    assert len(V.concat_gops(gops, 20)) == 20
    with pytest.raises(ValueError):
        V.segment_gops([])


def test_token_grid_and_wire_size():
    assert C.token_grid_shape(60, 50) == (8, 7)
    assert C.token_grid_shape(360, 640) == (45, 80)
    assert C.token_grid_shape(540, 960) == (68, 120)
    assert T.token_packet_wire_size(80, 12) == 996
    assert T.token_packet_wire_size(8, 12, 0) == 27


def test_drop_rate_math():
    # selection.py:70-87; test_selection.py:122-127
    assert S.drop_count(0.0, 3600) == 0
    assert S.drop_count(0.10, 3600) == 360
    assert S.drop_count(0.30, 3600) == 1080
    assert S.drop_count(0.25, 64) == 16
    with pytest.raises(ValueError):
        S.drop_count(0.31, 10)
    with pytest.raises(ValueError):
        S.drop_count(-0.1, 10)
    assert S.drop_rate_for_bandwidth(1000.0, 1000.0) == 0.0
    assert S.drop_rate_for_bandwidth(800.0, 1000.0) == pytest.approx(0.2)
    assert S.drop_rate_for_bandwidth(500.0, 1000.0) == S.DROP_RATE_CAP
    with pytest.raises(ValueError):
        S.drop_rate_for_bandwidth(500.0, 0.0)


def test_similarity_map_validation():
    with pytest.raises(ValueError):
        S.SimilarityMap(np.zeros(3))
    with pytest.raises(ValueError):
        S.SimilarityMap(np.full((2, 2), 1.5))
    m = S.SimilarityMap(np.full((2, 2), 1.0 + 1e-12))
    assert m.values.max() == 1.0


def test_errors_raised_before_any_device_work():
    tm = C.TokenMatrix("I", np.zeros((2, 2, 12)), np.ones((2, 2), bool))
    tp = C.TokenMatrix("P", np.zeros((2, 3, 12)), np.ones((2, 3), bool))
    with pytest.raises(ValueError):
        S.token_similarity(tm, tm)                       # kinds
    with pytest.raises(ValueError):
        S.token_similarity(tp, tm)                       # shapes
    with pytest.raises(ValueError):
        C.decode_gop(tm, tp, C.CodecConfig())            # shape mismatch
    with pytest.raises(ValueError):
        S.top_k_drop_mask(S.SimilarityMap(np.zeros((2, 2))), 5)
    with pytest.raises(ValueError, match="16-bit"):
        T.packetize_tokens(C.TokenMatrix("I", np.zeros((70_000, 1, 1)), np.ones((70_000, 1), bool)))
    f = V.Frame(np.zeros((8, 8, 3), np.float32))
    with pytest.raises(ValueError):
        C.downscale_frame(f, 1)
    with pytest.raises(ValueError):
        C.upscale_frame(f, 4)
    g = V.GoP(0, (f,) * 9)
    with pytest.raises(ValueError):
        C.scale_gop(g, 2, "sideways")
    with pytest.raises(ValueError):
        C.blend_boundary(g, g, 10)
    with pytest.raises(ValueError):
        C.blend_boundary(g, g, 0)
    pk = T.TokenPacket("P", 1, 0, 2, 12, 1, 0.0, 0.0, np.zeros(2, bool), b"")
    with pytest.raises(ValueError):
        T.reassemble([pk], (2, 2, 12), "P", gop_id=0)    # foreign gop_id


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    f = V.Frame(np.zeros((16, 16, 3), np.float32))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        C.encode_gop(V.GoP(0, (f,) * 9), C.CodecConfig())
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        C.downscale_frame(f, 2)


def test_public_names_mirror_reference_hot_path():
    # pkg/src/semstream/__init__.py:6-24 (hot-path subset) + module-level API
    for name in ("CodecConfig", "Frame", "GoP", "SimilarityMap", "TokenMatrix", "TokenPacket",
                 "blend_boundary", "boundary_flicker", "build_drop_mask", "decode_gop",
                 "downscale_frame", "drop_rate_for_bandwidth", "encode_gop", "packetize_tokens",
                 "psnr", "reassemble", "segment_gops", "token_similarity", "upscale_frame"):
        assert hasattr(P, name), name
    for mod, names in ((C, ("scale_gop", "apply_token_mask", "token_grid_shape",
                            "bilinear_upscale", "BLOCK", "COEFF_POSITIONS")),
                       (S, ("top_k_drop_mask", "DROP_RATE_CAP", "LOSS_TOLERANCE")),
                       (T, ("parse_packet", "token_packet_wire_size", "PacketFormatError"))):
        for n in names:
            assert hasattr(mod, n), n
    assert issubclass(T.PacketFormatError, ValueError)


def test_residual_packet_header_roundtrip():
    """Stream-file residual packets (transport.py:116-127,186-194): host-side
    header + CRC framing round trip and validation."""
    from paper_2602_03529_b200 import streamfile as SF
    pkt = SF.ResidualPacket(gop_id=7, theta=0.02, quant_step=1 / 127, window_length=9,
                            payload=b"\x01\x02\x03")
    data = pkt.to_bytes()
    assert data[:4] == b"\x4d\x53\x01\x02" and len(data) == 21 + 3 + 4   # >HBBIffBI = 21 B
    back = SF._parse_residual(data)
    assert back.gop_id == 7 and back.window_length == 9 and back.payload == b"\x01\x02\x03"
    bad = bytearray(data)
    bad[-5] ^= 1
    import pytest as _pt
    with _pt.raises(ValueError, match="crc"):
        SF._parse_residual(bytes(bad))
