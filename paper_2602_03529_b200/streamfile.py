"""The reference's stream-file container: the data format
on either side of the codec path for offline use, `semstream encode` /
`semstream decode` (cli.py:34-35, 67-74, 77-190), on the B200 path.

Layout (cli.py:34-35, 67-74): b"SMST" + version byte 1, then for every GoP
its I token packets (rows 0..H'-1), its P token packets, and optionally one
residual packet, each prefixed by its length as a big-endian u32.  The JSON
sidecar (video.py:217-230) carries the geometry and codec settings.

Every numeric stage runs through this package's drop-in API, i.e. on the
GPU: downscale + tokenize (K1), similarity + drop (K2), quantise + serialise
+ CRC (K3), parse + reassemble (K4), decode, residual (f1) and range coder
(f2), upscale + blend (K5).  The container framing, the residual packet
header (transport.py:45,116-127,186-194) and the JSON sidecar are host-side
byte handling, as in the reference.  Output bytes are identical to the
reference CLI's (tests/golden/stream_golden.json).
"""

from __future__ import annotations

import json
import struct
import zlib
from dataclasses import dataclass

import numpy as np

from . import residual as residual_mod
from .codec import (CodecConfig, apply_token_mask, blend_boundary, decode_gop, encode_gop,
                    scale_gop, token_grid_shape)
from .selection import build_drop_mask, token_similarity
from .transport import (KIND_RESIDUAL, MAGIC, VERSION, PacketFormatError, packetize_tokens,
                        parse_packet, reassemble)
from .video import GOP_SIZE, Frame, segment_gops

STREAM_MAGIC = b"SMST"            # cli.py:34
STREAM_VERSION = 1                # cli.py:35
_RESIDUAL_HDR = struct.Struct(">HBBIffBI")   # transport.py:45


class StreamFormatError(ValueError):
    """Malformed stream container (the reference CLI's CliError cases)."""


@dataclass(frozen=True)
class ResidualPacket:
    """transport.py:116-127."""

    gop_id: int
    theta: float
    quant_step: float
    window_length: int
    payload: bytes

    def to_bytes(self) -> bytes:
        body = _RESIDUAL_HDR.pack(MAGIC, VERSION, KIND_RESIDUAL, self.gop_id, self.theta,
                                  self.quant_step, self.window_length, len(self.payload))
        body += self.payload
        return body + struct.pack(">I", zlib.crc32(body) & 0xFFFFFFFF)


def _parse_residual(data: bytes) -> ResidualPacket:
    """transport.py:64-70 (seal) + 186-194 (residual branch)."""
    if len(data) < 4:
        raise PacketFormatError("packet shorter than its checksum")
    body, (crc,) = data[:-4], struct.unpack(">I", data[-4:])
    if zlib.crc32(body) & 0xFFFFFFFF != crc:
        raise PacketFormatError("crc32 mismatch")
    if len(body) < _RESIDUAL_HDR.size:
        raise PacketFormatError("residual packet header truncated")
    _, _, _, gop_id, theta, qstep, window, plen = _RESIDUAL_HDR.unpack(body[:_RESIDUAL_HDR.size])
    payload = body[_RESIDUAL_HDR.size:]
    if len(payload) != plen:
        raise PacketFormatError(f"residual payload length {len(payload)} != {plen}")
    return ResidualPacket(gop_id, theta, qstep, window, payload)


def parse_stream_packet(data: bytes):
    """parse_packet for the kinds a stream file holds: token packets through
    the GPU parser, residual packets through the host header parser."""
    if len(data) >= 8 and data[3] == KIND_RESIDUAL and \
            struct.unpack(">HB", data[:3]) == (MAGIC, VERSION):
        return _parse_residual(data)
    return parse_packet(data)


def _frame_block(packets) -> bytes:
    out = bytearray()
    for pkt in packets:
        data = pkt.to_bytes()
        out += struct.pack(">I", len(data)) + data
    return bytes(out)


def metadata(width: int, height: int, fps: float, frame_count: int, scale: int,
             extra: dict | None = None) -> str:
    """The JSON sidecar text (video.py:217-230: sort_keys, compact)."""
    meta = {"width": width, "height": height, "fps": fps, "frame_count": frame_count,
            "scale": scale}
    if extra:
        meta["codec"] = dict(extra)
    return json.dumps(meta, sort_keys=True, separators=(",", ":"))


def encode_clip(frames, scale: int = 2, fps: float = 30.0, theta: float = residual_mod.DEFAULT_THETA,
                drop_rate: float = 0.0, blend_width: int = 2, residual: bool = True):
    """`semstream encode` (cli.py:77-120) of a frame sequence.

    frames: iterable of Frame or (H, W, 3) float32 arrays.  Returns
    (stream bytes, sidecar JSON text)."""
    frames = [f if isinstance(f, Frame) else Frame(np.asarray(f, dtype=np.float32),
                                                   timestamp_index=t)
              for t, f in enumerate(frames)]
    if not frames:
        raise ValueError("empty frame sequence")
    cfg = CodecConfig(scale=scale, blend_width=blend_width)
    height, width = frames[0].height, frames[0].width
    meta = metadata(width, height, fps, len(frames), scale,
                    extra={"channels": cfg.channels, "theta": theta,
                           "quant_step": residual_mod.DEFAULT_QUANT_STEP,
                           "blend_width": blend_width, "drop_rate": drop_rate})
    out = bytearray(STREAM_MAGIC + bytes([STREAM_VERSION]))
    for k, gop in enumerate(segment_gops(frames)):
        working = scale_gop(gop, scale, "down")
        i_tokens, p_tokens = encode_gop(working, cfg)
        if drop_rate > 0.0:
            sim = token_similarity(p_tokens, i_tokens)
            p_tokens = apply_token_mask(p_tokens, build_drop_mask(sim, drop_rate))
        packets_i = packetize_tokens(i_tokens, scale=scale)
        packets_p = packetize_tokens(p_tokens, scale=scale)
        out += _frame_block(packets_i + packets_p)
        if residual:
            shape = i_tokens.values.shape
            i_quant = reassemble(packets_i, shape, "I", gop_id=k,
                                 frame_shape=i_tokens.frame_shape)
            p_quant = reassemble(packets_p, shape, "P", gop_id=k,
                                 frame_shape=i_tokens.frame_shape)
            recon = decode_gop(i_quant, p_quant, cfg)
            r = residual_mod.compute_residual(working, recon)
            sr = residual_mod.sparsify_quantize(residual_mod.aggregate_residual(r), theta=theta,
                                                gop_id=k)
            if sr.entry_count:
                pkt = ResidualPacket(gop_id=k, theta=theta, quant_step=sr.quant_step,
                                     window_length=GOP_SIZE,
                                     payload=residual_mod.encode_payload(sr))
                out += _frame_block([pkt])
    return bytes(out), meta


def read_stream(data: bytes) -> list:
    """cli.py:123-138: container header check, length-prefixed packets."""
    if data[:5] != STREAM_MAGIC + bytes([STREAM_VERSION]):
        raise StreamFormatError("not a semstream stream file")
    pos, packets = 5, []
    while pos < len(data):
        if pos + 4 > len(data):
            raise StreamFormatError(f"truncated packet length at byte {pos}")
        (n,) = struct.unpack(">I", data[pos:pos + 4])
        pos += 4
        if pos + n > len(data):
            raise StreamFormatError(f"truncated packet at byte {pos}")
        packets.append(parse_stream_packet(data[pos:pos + n]))
        pos += n
    return packets


def decode_stream(data: bytes, meta) -> list:
    """`semstream decode` (cli.py:141-190): stream bytes + sidecar (dict or
    JSON text) -> the reconstructed Frames (frame_count of them)."""
    if isinstance(meta, str):
        meta = json.loads(meta)
    packets = read_stream(data)
    codec_meta = meta.get("codec", {})
    cfg = CodecConfig(scale=meta["scale"], blend_width=codec_meta.get("blend_width", 2))
    scale = meta["scale"]
    work_h, work_w = -(-meta["height"] // scale), -(-meta["width"] // scale)
    h_tok, w_tok = token_grid_shape(work_h, work_w)
    channels = codec_meta.get("channels", cfg.channels)
    by_gop: dict = {}
    for pkt in packets:
        by_gop.setdefault(pkt.gop_id, []).append(pkt)
    frames_out, prev = [], None
    for k in sorted(by_gop):
        group = by_gop[k]
        i_pkts = [p for p in group if getattr(p, "kind", "") == "I"]
        p_pkts = [p for p in group if getattr(p, "kind", "") == "P"]
        res_pkts = [p for p in group if isinstance(p, ResidualPacket)]
        i_tokens = reassemble(i_pkts, (h_tok, w_tok, channels), "I", gop_id=k,
                              frame_shape=(work_h, work_w))
        p_tokens = reassemble(p_pkts, (h_tok, w_tok, channels), "P", gop_id=k,
                              frame_shape=(work_h, work_w))
        recon = decode_gop(i_tokens, p_tokens, cfg)
        if res_pkts:
            rp = res_pkts[0]
            sr = residual_mod.decode_payload(rp.payload, (work_h, work_w, 3), rp.theta,
                                             rp.quant_step, rp.window_length, gop_id=k)
            recon = residual_mod.apply_residual(recon, sr)
        recon = scale_gop(recon, scale, "up", crop=(meta["height"], meta["width"]))
        if prev is not None:
            recon = blend_boundary(prev, recon, cfg.blend_width)
        prev = recon
        frames_out.extend(recon.frames)
    return frames_out[:meta["frame_count"]]


def raw_rgb24(frames) -> bytes:
    """write_raw_video's bytes (video.py:139-143): rint(x * 255) as uint8."""
    return b"".join(np.rint(f.samples * 255.0).astype(np.uint8).tobytes() for f in frames)
