"""Token wire format -- drop-in for the token-packet half of
``semstream.transport`` (reference pkg/src/semstream/transport.py:1-305).

Packetisation (quantise + header + mask + payload + CRC-32), parsing /
validation and first-wins reassembly run on the GPU (``sst_packetize``,
``sst_serialize``, ``sst_parse``, ``sst_reassemble``); the bytes are identical
to the reference's ``TokenPacket.to_bytes()``.

Out of scope: residual / nack / bandwidth-report packets and the
receiver's GopAssembly / loss policy (control plane).  ``parse_packet``
rejects those kinds with ``PacketFormatError``.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _dev, _lib
from .codec import TokenMatrix

MAGIC = 0x4D53            # transport.py:32
VERSION = 1               # transport.py:33
KIND_I = 0                # transport.py:35
KIND_P = 1
KIND_RESIDUAL = 2
KIND_NACK = 3
KIND_BW_REPORT = 4

_KIND_TO_NAME = {KIND_I: "I", KIND_P: "P"}
_NAME_TO_KIND = {"I": KIND_I, "P": KIND_P}
_TOKEN_HDR = struct.Struct(">HBBIHHBBff")     # transport.py:44 (22 bytes)


class PacketFormatError(ValueError):
    """Packet bytes failed structural or checksum validation (transport.py:52-53)."""


def token_packet_wire_size(width_tokens: int, channels: int, valid_count: int | None = None) -> int:
    """transport.py:221-226."""
    if valid_count is None:
        valid_count = width_tokens
    return _TOKEN_HDR.size + (width_tokens + 7) // 8 + valid_count * channels + 4


def _round16(n: int) -> int:
    return (n + 15) & ~15


@dataclass(frozen=True)
class TokenPacket:
    """One token row with its position mask and 8-bit payload (transport.py:82-112)."""

    kind: str
    gop_id: int
    row_index: int
    width_tokens: int
    channels: int
    scale: int
    quant_min: float
    quant_range: float
    mask: np.ndarray
    payload: bytes
    _wire: bytes | None = field(default=None, compare=False, repr=False)

    def to_bytes(self) -> bytes:
        """Sealed wire bytes (transport.py:97-102)."""
        if self._wire is not None:
            return self._wire
        return serialize_packets([self])[0]

    @property
    def valid_count(self) -> int:
        return int(np.count_nonzero(self.mask))

    def dequantized(self) -> np.ndarray:
        """(valid_count, C) token vectors recovered from the payload
        (transport.py:108-112), dequantised on the GPU."""
        probe = replace(self, row_index=0, _wire=None)
        width = len(self.mask)
        m = reassemble([probe], (1, width, self.channels), self.kind, self.gop_id)
        return m.values[0][np.asarray(self.mask, bool)]


# ---------------------------------------------------------------------------
# device batches of packet fields

def _field_batch(packets) -> tuple:
    """SstPacketInfo records + concatenated (mask bits | payload) bytes."""
    n = len(packets)
    info = np.zeros(n, dtype=_lib.INFO_DTYPE)
    chunks = []
    offs = np.zeros(n, dtype=np.int64)
    pos = 0
    for j, p in enumerate(packets):
        mask = np.asarray(p.mask, dtype=bool)
        mbytes = np.packbits(mask.astype(np.uint8)).tobytes()
        payload = bytes(p.payload)
        rec = info[j]
        rec["kind"] = _NAME_TO_KIND[p.kind]
        rec["gop_id"] = p.gop_id
        rec["row"] = p.row_index
        rec["width"] = len(mask)
        rec["channels"] = p.channels
        rec["scale"] = p.scale
        rec["valid"] = int(mask.sum())
        rec["qmin"] = np.float32(p.quant_min)
        rec["qrange"] = np.float32(p.quant_range)
        rec["dqmin"] = float(p.quant_min)
        rec["dqrange"] = float(p.quant_range)
        rec["mask_off"] = 0
        rec["payload_off"] = len(mbytes)
        offs[j] = pos
        blob = mbytes + payload
        chunks.append(blob)
        pos += len(blob)
    buf = np.frombuffer(b"".join(chunks) or b"\0", dtype=np.uint8)
    return info, buf, offs


def serialize_packets(packets) -> list:
    """TokenPacket.to_bytes for many field-wise packets in one GPU launch.
    Like the reference, the payload is serialised exactly as given."""
    packets = list(packets)
    if not packets:
        return []
    for p in packets:
        if p.kind not in _NAME_TO_KIND:
            raise KeyError(p.kind)
        if (p.channels == 0 and len(p.payload)) or (p.channels and len(p.payload) % p.channels):
            raise ValueError("payload length is not a multiple of the channel count")
    info, buf, offs = _field_batch(packets)
    for j, p in enumerate(packets):
        info[j]["valid"] = len(p.payload) // p.channels if p.channels else 0
    sizes = np.array([_TOKEN_HDR.size + (len(p.mask) + 7) // 8 + len(p.payload) + 4
                      for p in packets], dtype=np.int64)
    if int(sizes.max()) > 48 * 1024:
        raise ValueError("token packet larger than the 48 KiB serialiser staging limit")
    out_off = np.zeros(len(packets), dtype=np.int64)
    out_off[1:] = np.cumsum(sizes)[:-1]
    d_info = _dev.h2d(info.view(np.uint8))
    d_buf = _dev.h2d(buf)
    d_moff = _dev.h2d(offs)
    d_poff = _dev.h2d(offs + info["payload_off"].astype(np.int64))
    d_out = _dev.empty((int(sizes.sum()),), torch.uint8)
    d_ooff = _dev.h2d(out_off)
    _lib.call("sst_serialize", _dev.ptr(d_info), _dev.ptr(d_buf), _dev.ptr(d_moff), _dev.ptr(d_buf),
              _dev.ptr(d_poff), len(packets), _dev.ptr(d_out), _dev.ptr(d_ooff), _dev.stream())
    raw = _dev.d2h(d_out).tobytes()
    return [raw[o:o + s] for o, s in zip(out_off.tolist(), sizes.tolist())]


# ---------------------------------------------------------------------------
# packetisation

def packetize_tokens(m: TokenMatrix, scale: int = 1) -> list:
    """One packet per token row, header-only rows included (transport.py:236-271)."""
    h = m.height_tokens
    if h > 0xFFFF:
        raise ValueError(f"matrix has {h} rows; the row index field is 16-bit")
    if h == 0:
        return []
    w, c = m.width_tokens, m.channels
    slot = _round16(token_packet_wire_size(w, c, w))
    vals = _dev.h2d(m.values, np.float64)
    mask = _dev.h2d(m.mask, np.uint8)
    kind = _dev.h2d(np.array([_NAME_TO_KIND[m.kind]], np.uint8))
    gop = _dev.h2d(np.array([m.gop_id], np.uint32))
    sc = _dev.h2d(np.array([scale], np.uint8))
    arena = _dev.empty((h, slot), torch.uint8)
    lengths = _dev.empty((h,), torch.int32)
    _lib.call("sst_packetize", _dev.ptr(vals), _dev.ptr(mask), 1, h, w, c, _dev.ptr(kind),
              _dev.ptr(gop), _dev.ptr(sc), _dev.ptr(arena), slot, _dev.ptr(lengths), _dev.stream())
    return _packets_from_arena(_dev.d2h(arena), _dev.d2h(lengths), m.mask, m.kind)


def _packets_from_arena(arena: np.ndarray, lengths: np.ndarray, masks: np.ndarray, kind: str):
    out = []
    for r in range(arena.shape[0]):
        data = arena[r, :int(lengths[r])].tobytes()
        (_, _, _, gop_id, row, width, channels, scale, qmin, qrange) = \
            _TOKEN_HDR.unpack_from(data, 0)
        mlen = (width + 7) // 8
        out.append(TokenPacket(kind=kind, gop_id=gop_id, row_index=row, width_tokens=width,
                               channels=channels, scale=scale, quant_min=qmin,
                               quant_range=qrange, mask=np.array(masks[r], dtype=bool),
                               payload=data[_TOKEN_HDR.size + mlen:-4], _wire=data))
    return out


# ---------------------------------------------------------------------------
# parsing

def _format_error(status: int, data: bytes, rec) -> PacketFormatError:
    if status == _lib.PKT_SHORT:
        return PacketFormatError("packet shorter than its checksum")
    if status == _lib.PKT_CRC:
        return PacketFormatError("crc32 mismatch")
    if status == _lib.PKT_BODY_SHORT:
        return PacketFormatError("packet body too short")
    if status == _lib.PKT_MAGIC:
        return PacketFormatError(f"bad magic 0x{struct.unpack('>H', data[:2])[0]:04X}")
    if status == _lib.PKT_VERSION:
        return PacketFormatError(f"unsupported version {data[2]}")
    if status == _lib.PKT_KIND:
        kind = int(rec["kind"])
        if kind in (KIND_RESIDUAL, KIND_NACK, KIND_BW_REPORT):
            return PacketFormatError(
                f"packet kind {kind} is a control / residual packet, outside the codec path")
        return PacketFormatError(f"unknown packet kind {kind}")
    if status == _lib.PKT_HDR_TRUNC:
        return PacketFormatError("token packet header truncated")
    if status == _lib.PKT_MASK_TRUNC:
        return PacketFormatError("token packet mask truncated")
    if status == _lib.PKT_PAYLOAD_LEN:
        plen = len(data) - 4 - int(rec["payload_off"])
        return PacketFormatError(
            f"payload length {plen} != popcount(mask)*C = {int(rec['valid']) * int(rec['channels'])}")
    if status == _lib.PKT_NEG_RANGE:
        return PacketFormatError("negative quantization range")
    return PacketFormatError(f"packet rejected (status {status})")


def parse_packets(datas, errors: str = "raise") -> list:
    """Batched parse_packet: one GPU launch validates every packet.
    errors='raise' raises on the first bad packet (reference order);
    errors='none' returns None in its place."""
    datas = [bytes(d) for d in datas]
    n = len(datas)
    if n == 0:
        return []
    lens = np.array([len(d) for d in datas], dtype=np.int32)
    offs = np.zeros(n, dtype=np.int64)
    offs[1:] = np.cumsum(lens.astype(np.int64))[:-1]
    buf = np.frombuffer(b"".join(datas) or b"\0", dtype=np.uint8)
    d_buf = _dev.h2d(buf)
    d_off = _dev.h2d(offs)
    d_len = _dev.h2d(lens)
    d_info = _dev.empty((n * _lib.INFO_BYTES,), torch.uint8)
    _lib.call("sst_parse", _dev.ptr(d_buf), _dev.ptr(d_off), _dev.ptr(d_len), None, n,
              _dev.ptr(d_info), _dev.stream())
    info = _dev.d2h(d_info).view(_lib.INFO_DTYPE)
    out = []
    for j, data in enumerate(datas):
        rec = info[j]
        st = int(rec["status"])
        if st != _lib.PKT_OK:
            if errors == "raise":
                raise _format_error(st, data, rec)
            out.append(None)
            continue
        width = int(rec["width"])
        moff, poff = int(rec["mask_off"]), int(rec["payload_off"])
        bits = np.unpackbits(np.frombuffer(data[moff:poff], dtype=np.uint8))
        out.append(TokenPacket(kind=_KIND_TO_NAME[int(rec["kind"])], gop_id=int(rec["gop_id"]),
                               row_index=int(rec["row"]), width_tokens=width,
                               channels=int(rec["channels"]), scale=int(rec["scale"]),
                               quant_min=float(rec["qmin"]), quant_range=float(rec["qrange"]),
                               mask=bits[:width].astype(bool), payload=data[poff:-4],
                               _wire=data))
    return out


def parse_packet(data: bytes):
    """Parse one wire packet, validating checksum, magic, version and
    lengths (transport.py:154-218)."""
    return parse_packets([data])[0]


# ---------------------------------------------------------------------------
# reassembly

def reassemble(packets, expected: tuple, kind: str, gop_id: int = 0,
               frame_shape: tuple | None = None, stats: dict | None = None) -> TokenMatrix:
    """Zero-fill, first-arrival-wins reassembly (transport.py:274-305)."""
    h, w, c = expected
    packets = list(packets)
    for pkt in packets:
        if pkt.kind != kind or pkt.gop_id != gop_id:
            raise ValueError(f"packet ({pkt.kind}, gop {pkt.gop_id}) does not belong to "
                             f"({kind}, gop {gop_id})")
    # The rows the reference dequantises (in range, first arrival, any valid
    # column) must carry popcount(mask) * C payload bytes: TokenPacket.dequantized
    # reshapes the payload and raises ValueError otherwise (transport.py:108-112,
    # 292-301).  The kernel trusts these lengths, so check them here.
    seen = set()
    for pkt in packets:
        if pkt.row_index >= h or pkt.row_index in seen:
            continue
        seen.add(pkt.row_index)
        pmask = np.asarray(pkt.mask, dtype=bool)
        if pmask[:w].any():
            need = int(np.count_nonzero(pmask)) * int(pkt.channels)
            if len(pkt.payload) != need:
                raise ValueError(f"cannot reshape array of size {len(pkt.payload)} into shape "
                                 f"({int(np.count_nonzero(pmask))},{pkt.channels})")
    n = len(packets)
    values = _dev.empty((h, w, c), torch.float64)
    mask = _dev.empty((h, w), torch.uint8)
    winner = _dev.empty((max(h, 1),), torch.int32)
    d_stats = _dev.empty((2,), torch.int32)
    exp_kind = _dev.h2d(np.array([_NAME_TO_KIND[kind]], np.uint8))
    exp_gop = _dev.h2d(np.array([gop_id & 0xFFFFFFFF], np.uint32))
    d_info = d_buf = d_off = d_target = None
    if n:
        info, buf, offs = _field_batch(packets)
        d_info = _dev.h2d(info.view(np.uint8))
        d_buf = _dev.h2d(buf)
        d_off = _dev.h2d(offs)
        d_target = _dev.zeros((n,), torch.int32)
    _lib.call("sst_reassemble", _dev.ptr(d_buf), _dev.ptr(d_off), _dev.ptr(d_info),
              _dev.ptr(d_target), n, 1, h, w, c, _dev.ptr(exp_kind), _dev.ptr(exp_gop),
              _dev.ptr(winner), _dev.ptr(values), _dev.ptr(mask), _dev.ptr(d_stats),
              _dev.stream())
    if n:
        st = _dev.d2h(d_info).view(_lib.INFO_DTYPE)["status"]
        bad = np.flatnonzero(st == _lib.PKT_SHAPE)
        if bad.size:
            p = packets[int(bad[0])]
            raise ValueError(f"packet row {p.row_index} (width {len(p.mask)}, "
                             f"{p.channels} channels) does not fit a {expected} matrix")
    corrupt, rows = (int(v) for v in _dev.d2h(d_stats))
    if stats is not None:
        if corrupt:
            stats["corrupt"] = stats.get("corrupt", 0) + corrupt
        stats["rows_received"] = rows
    return TokenMatrix(kind, _dev.d2h(values), _dev.d2h(mask).astype(bool), gop_id=gop_id,
                       frame_shape=frame_shape)
