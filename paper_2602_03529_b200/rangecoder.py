"""Adaptive range coding of sparse-residual scans -- drop-in for
``semstream.rangecoder`` (reference pkg/src/semstream/rangecoder.py).

Encoding and decoding run on the GPU (csrc/residual.cu: one CTA per stream,
parallel non-zero compaction, serial carry-less coder with a Fenwick-tree
model); many streams are coded concurrently.  The symbol-mapping helpers are
scalar host utilities, as in the reference.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib

EOS = 0                 # rangecoder.py:21-23
MAX_RUN = 255
ALPHABET_SIZE = 510

_STATUS = {1: "compressed stream truncated", 2: "zero run overruns scan length",
           3: "value overruns scan length", 4: "symbol budget exceeded before EOS",
           5: "EOS before end of stream", 6: "symbol stream missing EOS"}


class CorruptStreamError(ValueError):
    """Compressed bytes are truncated or otherwise undecodable (rangecoder.py:32-33)."""


def zero_run_symbol(k: int) -> int:
    if not 1 <= k <= MAX_RUN:
        raise ValueError(f"zero-run length must be in [1, {MAX_RUN}], got {k}")
    return k


def value_symbol(v: int) -> int:
    if v == 0 or not -127 <= v <= 127:
        raise ValueError(f"value symbol must be nonzero in [-127, 127], got {v}")
    return v + 383 if v < 0 else v + 382


def symbol_kind(sym: int):
    if sym == EOS:
        return "eos", None
    if 1 <= sym <= MAX_RUN:
        return "run", sym
    if 256 <= sym <= 382:
        return "value", sym - 383
    if 383 <= sym < ALPHABET_SIZE:
        return "value", sym - 382
    raise ValueError(f"symbol id {sym} outside alphabet")


def validate_stream(symbols) -> None:
    if not len(symbols):
        raise ValueError("symbol stream must end with EOS")
    for i, sym in enumerate(symbols):
        kind, _ = symbol_kind(int(sym))
        if kind == "eos" and i != len(symbols) - 1:
            raise ValueError(f"EOS at position {i} before end of stream")
    if int(symbols[-1]) != EOS:
        raise ValueError("symbol stream must end with EOS")


def scan_to_symbols(dense) -> list:
    """Zero runs + values + EOS for a dense scan (rangecoder.py:75-94)."""
    dense = np.asarray(dense)
    nz = np.flatnonzero(dense)
    out = []
    pos = 0
    for idx in nz.tolist():
        gap = idx - pos
        out.extend([MAX_RUN] * (gap // MAX_RUN))
        if gap % MAX_RUN:
            out.append(gap % MAX_RUN)
        out.append(value_symbol(int(dense[idx])))
        pos = idx + 1
    out.append(EOS)
    return out


def symbols_to_scan(symbols, length: int) -> np.ndarray:
    """rangecoder.py:97-116."""
    out = np.zeros(length, dtype=np.int16)
    pos = 0
    for i, sym in enumerate(symbols):
        kind, arg = symbol_kind(int(sym))
        if kind == "eos":
            if i != len(symbols) - 1:
                raise CorruptStreamError(f"EOS at position {i} before end of stream")
            return out
        if kind == "run":
            pos += arg
            if pos > length:
                raise CorruptStreamError(f"zero run overruns scan length {length}")
        else:
            if pos >= length:
                raise CorruptStreamError(f"value overruns scan length {length}")
            out[pos] = arg
            pos += 1
    raise CorruptStreamError("symbol stream missing EOS")


# ---------------------------------------------------------------------------
# device coding

def _encode_dev(scans: torch.Tensor, G: int, n: int) -> list:
    """scans: device int16 [G*n]; returns G payloads."""
    cap = max(64, n // 2 + 64)
    while True:
        idx = _dev.empty((max(G * n, 1),), torch.int64)
        out = _dev.empty((G * cap,), torch.uint8)
        olen = _dev.empty((G,), torch.int64)
        _lib.call("sst_rc_encode", _dev.ptr(scans), G, n, _dev.ptr(idx), _dev.ptr(out), cap,
                  _dev.ptr(olen), _dev.stream())
        lens = _dev.d2h(olen)
        if (lens >= 0).all():
            raw = _dev.d2h(out)
            return [raw[g * cap:g * cap + int(lens[g])].tobytes() for g in range(G)]
        cap = int(-lens.min()) + 64


def encode_dense_device(scan: torch.Tensor) -> bytes:
    """encode_scan of one device-resident int16 scan."""
    return _encode_dev(scan, 1, scan.numel())[0]


def encode_scans(scans) -> list:
    """encode_scan for many equal-length scans in one launch (one CTA each)."""
    arr = np.stack([np.asarray(s, dtype=np.int16).ravel() for s in scans])
    G, n = arr.shape
    return _encode_dev(_dev.h2d(arr.ravel()), G, n)


def encode_scan(dense) -> bytes:
    """rangecoder.py:238-239."""
    return encode_scans([dense])[0]


def decode_scans(datas, length: int) -> list:
    """decode_scan for many payloads in one launch."""
    datas = [bytes(d) for d in datas]
    G = len(datas)
    lens = np.array([len(d) for d in datas], dtype=np.int64)
    offs = np.zeros(G, dtype=np.int64)
    offs[1:] = np.cumsum(lens)[:-1]
    buf = _dev.h2d(np.frombuffer(b"".join(datas) or b"\0", dtype=np.uint8))
    scans = _dev.empty((max(G * length, 1),), torch.int16)
    status = _dev.empty((G,), torch.int32)
    d_off, d_len = _dev.h2d(offs), _dev.h2d(lens)     # keep alive until the launch is queued
    _lib.call("sst_rc_decode", _dev.ptr(buf), _dev.ptr(d_off), _dev.ptr(d_len), G, length,
              _dev.ptr(scans), _dev.ptr(status), _dev.stream())
    st = _dev.d2h(status)
    for g in range(G):
        if st[g]:
            raise CorruptStreamError(_STATUS.get(int(st[g]), f"undecodable stream ({st[g]})"))
    out = _dev.d2h(scans[:G * length]) if length else np.zeros(0, np.int16)
    return [out[g * length:(g + 1) * length].copy() for g in range(G)]


def decode_scan(data: bytes, length: int) -> np.ndarray:
    """rangecoder.py:242-243."""
    return decode_scans([data], length)[0]


def encode_stream(symbols) -> bytes:
    """Encode a validated symbol stream (rangecoder.py:155-185).  Streams that
    are the canonical symbolisation of a scan go straight to the device coder;
    others (e.g. split zero runs) through the symbol-list kernel."""
    validate_stream(symbols)
    syms = np.asarray(symbols, dtype=np.int32)
    return encode_symbol_streams([syms])[0]


def encode_symbol_streams(streams) -> list:
    streams = [np.asarray(s, dtype=np.int32) for s in streams]
    G = len(streams)
    lens = np.array([len(s) for s in streams], dtype=np.int64)
    offs = np.zeros(G, dtype=np.int64)
    offs[1:] = np.cumsum(lens)[:-1]
    d_syms = _dev.h2d(np.concatenate(streams) if G else np.zeros(1, np.int32))
    cap = int(max(64, 2 * lens.max() + 64)) if G else 64
    d_off, d_len = _dev.h2d(offs), _dev.h2d(lens)
    while True:
        out = _dev.empty((max(G * cap, 1),), torch.uint8)
        olen = _dev.empty((max(G, 1),), torch.int64)
        _lib.call("sst_rc_encode_symbols", _dev.ptr(d_syms), _dev.ptr(d_off), _dev.ptr(d_len), G,
                  _dev.ptr(out), cap, _dev.ptr(olen), _dev.stream())
        ol = _dev.d2h(olen)[:G]
        if (ol >= 0).all():          # a negative length is the size the output needed
            raw = _dev.d2h(out)
            return [raw[g * cap:g * cap + int(ol[g])].tobytes() for g in range(G)]
        cap = int(-ol.min()) + 64


def decode_stream(data: bytes, max_symbols: int = 1 << 24) -> list:
    """Decode to the exact symbol list (rangecoder.py:188-235)."""
    data = bytes(data)
    # The adaptive model can code a symbol in well under one bit, so the byte
    # count does not bound the symbol count: start from a guess and grow the
    # output on status 7 (capacity exceeded) up to the caller's budget.
    cap = max(1, min(max_symbols, max(16, 8 * len(data) + 16)))
    buf = _dev.h2d(np.frombuffer(data or b"\0", dtype=np.uint8))
    nsym = _dev.empty((1,), torch.int64)
    status = _dev.empty((1,), torch.int32)
    while True:
        syms = _dev.empty((cap,), torch.int32)
        _lib.call("sst_rc_decode_symbols", _dev.ptr(buf), len(data), max_symbols, cap,
                  _dev.ptr(syms), _dev.ptr(nsym), _dev.ptr(status), _dev.stream())
        st = int(status.item())
        if st != 7 or cap >= max_symbols:
            break
        cap = min(max_symbols, cap * 8)
    if st == 1:
        raise CorruptStreamError(f"compressed stream truncated ({len(data)} bytes)")
    if st == 4:
        raise CorruptStreamError("symbol budget exceeded before EOS")
    if st:
        raise CorruptStreamError(_STATUS.get(st, f"undecodable stream ({st})"))
    return [int(s) for s in _dev.d2h(syms[:int(nsym.item())])]
