"""ORACLE / TEST INFRASTRUCTURE ONLY.

CPU restatement (numpy, float64 where the reference is float64) of the
reference codec hot path, used as the parity checker by ``tests/``, by
``__graft_entry__.smoke()`` and as the CPU baseline leg of ``bench.py``.  The
product path (``paper_2602_03529_b200``) never imports this module.

Every function cites the reference ``file:line`` (relative to
``/root/reference/pkg/src/semstream``) whose arithmetic it restates.  The
restatement reproduces the reference's floating-point operation order so that
results are bit-identical, not merely close:

* box downscale: exact s x s sum in row-major window order, one correctly
  rounded division by s*s, cast to float32 (codec.py:202-214);
* P source: sequential float64 sum of frames 1..8 then /8 (codec.py:151-152);
* DCT / IDCT: the ducc0 algorithm restated in ``oracle/dct8.py``;
* similarity: numpy's pairwise summation order for 12 channels (8-way
  unrolled block then sequential tail) (selection.py:44-46);
* quantiser: float64 ``rint`` half-to-even on (v - qmin32) * (255/qrange32)
  (transport.py:248-266);
* bilinear: half-pixel centres, separate mul/add in the reference's order
  (codec.py:217-235);
* blend: alpha * prev + (1 - alpha) * curr in float64 (codec.py:289-293).

``clip`` follows numpy's ``np.clip`` semantics (x < lo -> lo, x > hi -> hi,
else x; -0.0 is kept).  Row min/max over signed zeros: numpy's SIMD reduction
returns a sign that depends on the host's vector width, so the reference has
no portable answer there; this oracle and the CUDA kernels both use the total
order -0.0 < +0.0 (documented in DESIGN.md).

Parity status: pinned.  See tests/test_oracle_reference.py (live reference,
container only) and tests/golden/ (fixtures generated from the reference by
tests/golden/make_golden.py).
"""

from __future__ import annotations

import struct
import zlib

import numpy as np

from .dct8 import dctn2_8x8, idctn2_8x8

GOP_SIZE = 9                                         # video.py:12
BLOCK = 8                                            # codec.py:20
COEFF_POSITIONS = ((0, 0), (0, 1), (1, 0), (2, 0))   # codec.py:22
CHANNELS = 12                                        # codec.py:32
PSNR_CAP_DB = 99.0                                   # video.py:13
LOSS_TOLERANCE = 0.30                                # selection.py:14
DROP_RATE_CAP = 0.25                                 # selection.py:13

MAGIC = 0x4D53                                       # transport.py:32
VERSION = 1                                          # transport.py:33
KIND_I, KIND_P = 0, 1                                # transport.py:35-36
TOKEN_HDR = struct.Struct(">HBBIHHBBff")             # transport.py:44
HDR_SIZE = TOKEN_HDR.size                            # 22 bytes


class OraclePacketError(ValueError):
    """Mirror of transport.PacketFormatError (transport.py:52-53)."""


# ---------------------------------------------------------------------------
# numpy-semantics helpers

def np_clip01(x: np.ndarray) -> np.ndarray:
    """np.clip(x, 0.0, 1.0) including the -0.0 pass-through."""
    return np.clip(x, 0.0, 1.0)


def row_min_max(vals: np.ndarray) -> tuple[float, float]:
    """Min / max with the canonical signed-zero order -0.0 < +0.0."""
    flat = np.asarray(vals, dtype=np.float64).ravel()
    mn = flat.min()
    mx = flat.max()
    if mn == 0.0:
        mn = -0.0 if np.any((flat == 0.0) & np.signbit(flat)) else 0.0
    if mx == 0.0:
        mx = 0.0 if np.any((flat == 0.0) & ~np.signbit(flat)) else -0.0
    return float(mn), float(mx)


# ---------------------------------------------------------------------------
# a4/a5: scaling geometry, box downscale

def working_shape(h: int, w: int, s: int) -> tuple[int, int]:
    """ceil(dim / s) (codec.py:209-212)."""
    return -(-h // s), -(-w // s)


def token_grid_shape(h: int, w: int) -> tuple[int, int]:
    """codec.py:94-96."""
    return -(-h // BLOCK), -(-w // BLOCK)


def downscale(frames: np.ndarray, s: int) -> np.ndarray:
    """Box downscale of (..., H, W, 3) float32 frames (codec.py:202-214).

    Edge-replicate to a multiple of s, sum each s x s window in row-major
    order in float64, divide once by s*s, round to float32.
    """
    if s not in (2, 3):
        raise ValueError(f"scale factor must be 2 or 3, got {s}")
    img = np.asarray(frames, dtype=np.float64)
    h, w = img.shape[-3:-1]
    ph, pw = (-h) % s, (-w) % s
    if ph or pw:
        pad = [(0, 0)] * (img.ndim - 3) + [(0, ph), (0, pw), (0, 0)]
        img = np.pad(img, pad, mode="edge")
    hh, ww = img.shape[-3] // s, img.shape[-2] // s
    v = img.reshape(img.shape[:-3] + (hh, s, ww, s, 3))
    acc = None
    for j in range(s):
        for l in range(s):
            term = v[..., :, j, :, l, :]
            acc = 0.0 + term if acc is None else acc + term   # numpy add.reduce starts at 0.0
    return (acc / float(s * s)).astype(np.float32)


# ---------------------------------------------------------------------------
# a6: tokenizer

def _pad_block(img: np.ndarray) -> np.ndarray:
    """Edge pad a working image to a multiple of 8 (codec.py:99-105)."""
    h, w = img.shape[:2]
    ph, pw = (-h) % BLOCK, (-w) % BLOCK
    if ph or pw:
        img = np.pad(img, ((0, ph), (0, pw), (0, 0)), mode="edge")
    return img


def tokenize(img: np.ndarray) -> np.ndarray:
    """(h, w, 3) image -> (H', W', 12) tokens (codec.py:120-128)."""
    img = _pad_block(np.asarray(img, dtype=np.float64))
    hb, wb = img.shape[0] // BLOCK, img.shape[1] // BLOCK
    blocks = img.reshape(hb, BLOCK, wb, BLOCK, 3).transpose(0, 2, 4, 1, 3)
    coeffs = dctn2_8x8(blocks)
    out = np.empty((hb, wb, 3, 4), dtype=np.float64)
    for k, (y, x) in enumerate(COEFF_POSITIONS):
        out[..., k] = coeffs[..., y, x]
    return out.reshape(hb, wb, CHANNELS)


def p_source(frames9: np.ndarray) -> np.ndarray:
    """Temporal mean of frames 1..8 in float64 (codec.py:151-152)."""
    acc = 0.0 + np.asarray(frames9[1], dtype=np.float64)    # add.reduce identity start
    for t in range(2, GOP_SIZE):
        acc = acc + np.asarray(frames9[t], dtype=np.float64)
    return acc / 8.0


def encode(frames9: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Working-res GoP (9, h, w, 3) f32 -> (I, P) token values (codec.py:143-157)."""
    if len(frames9) != GOP_SIZE:
        raise ValueError(f"GoP must hold {GOP_SIZE} frames")
    return tokenize(frames9[0]), tokenize(p_source(frames9))


# ---------------------------------------------------------------------------
# a8-a11: similarity, drop mask, mask application

def _pairwise12(x: np.ndarray) -> np.ndarray:
    """numpy pairwise-sum order for a 12-long contiguous axis."""
    r = ((x[..., 0] + x[..., 1]) + (x[..., 2] + x[..., 3])) + \
        ((x[..., 4] + x[..., 5]) + (x[..., 6] + x[..., 7]))
    for c in range(8, x.shape[-1]):
        r = r + x[..., c]
    return 0.0 + r                      # add.reduce: identity 0.0 + pairwise block


def _reduce_sum(x: np.ndarray) -> np.ndarray:
    if x.shape[-1] == CHANNELS:
        return _pairwise12(x)
    if x.shape[-1] < 8:                 # numpy: plain sequential loop from 0.0
        r = 0.0 + x[..., 0]
        for c in range(1, x.shape[-1]):
            r = r + x[..., c]
        return r
    return np.sum(x, axis=-1)           # other widths: defer to numpy itself


def similarity(p: np.ndarray, i: np.ndarray) -> np.ndarray:
    """Cosine similarity with zero-norm conventions (selection.py:33-52)."""
    p = np.asarray(p, dtype=np.float64)
    i = np.asarray(i, dtype=np.float64)
    dot = _reduce_sum(p * i)
    pn = np.sqrt(_reduce_sum(p * p))
    inorm = np.sqrt(_reduce_sum(i * i))
    denom = pn * inorm
    with np.errstate(invalid="ignore", divide="ignore"):
        sim = np.where(denom > 0.0, dot / np.where(denom > 0.0, denom, 1.0), 0.0)
    sim = np.where((pn == 0.0) & (inorm == 0.0), 1.0, sim)
    return np.clip(sim, -1.0, 1.0)


def drop_count(rate: float, n: int) -> int:
    """k = floor(rate * N + 0.5) with the tolerance check (selection.py:70-79)."""
    if rate < 0.0:
        raise ValueError(f"drop rate must be non-negative, got {rate}")
    if rate > LOSS_TOLERANCE:
        raise ValueError(f"drop rate {rate} exceeds the {LOSS_TOLERANCE} tolerance envelope")
    return int(np.floor(rate * n + 0.5))


def top_k_mask(sim: np.ndarray, k: int) -> np.ndarray:
    """k highest similarities, ties in row-major order (selection.py:55-67).

    Restated as a rank test instead of a sort: position j is dropped iff
    #{i : sim_i > sim_j} + #{i < j : sim_i == sim_j} < k.
    """
    flat = np.asarray(sim, dtype=np.float64).ravel()
    n = flat.size
    if not 0 <= k <= n:
        raise ValueError(f"k must be in [0, {n}], got {k}")
    mask = np.zeros(n, dtype=bool)
    if k:
        order = sorted(range(n), key=lambda j: (-flat[j], j))
        mask[np.array(order[:k], dtype=np.int64)] = True
    return mask.reshape(np.shape(sim))


def apply_mask(values: np.ndarray, mask: np.ndarray, drop: np.ndarray):
    """codec.py:189-196."""
    new_mask = np.asarray(mask, bool) & ~np.asarray(drop, bool)
    return np.where(new_mask[..., None], values, 0.0), new_mask


# ---------------------------------------------------------------------------
# a12-a15: wire format

def _crc(data: bytes) -> int:
    return zlib.crc32(data) & 0xFFFFFFFF          # transport.py:56-57


def quantize_row(vals: np.ndarray):
    """Per-row quantiser (transport.py:248-266): returns (qmin32, qrange32, payload)."""
    if vals.size == 0:
        return 0.0, 0.0, b""
    qmin, qmax = row_min_max(vals)
    qrange = qmax - qmin
    qmin32 = float(np.float32(qmin))
    qrange32 = float(np.float32(qrange))
    if qrange32 > 0.0:
        levels = np.rint((vals - qmin32) * (255.0 / qrange32))
        payload = np.clip(levels, 0, 255).astype(np.uint8).tobytes()
    else:
        payload = bytes(vals.size)
    return qmin32, qrange32, payload


def pack_row(kind: int, gop_id: int, row: int, values_row: np.ndarray,
             mask_row: np.ndarray, scale: int) -> bytes:
    """One token-row packet, sealed (transport.py:97-102, 236-271)."""
    width, channels = values_row.shape
    valid = values_row[np.asarray(mask_row, bool)]
    qmin32, qrange32, payload = quantize_row(valid)
    body = TOKEN_HDR.pack(MAGIC, VERSION, kind, gop_id, row, width, channels, scale,
                          qmin32, qrange32)
    body += np.packbits(np.asarray(mask_row, np.uint8)).tobytes() + payload
    return body + struct.pack(">I", _crc(body))


def packetize(kind: int, gop_id: int, values: np.ndarray, mask: np.ndarray,
              scale: int = 1) -> list[bytes]:
    """All rows of one token matrix (transport.py:236-271)."""
    h = values.shape[0]
    if h > 0xFFFF:
        raise ValueError(f"matrix has {h} rows; the row index field is 16-bit")
    return [pack_row(kind, gop_id, r, values[r], mask[r], scale) for r in range(h)]


def wire_size(width: int, channels: int, valid: int | None = None) -> int:
    """transport.py:221-226."""
    if valid is None:
        valid = width
    return HDR_SIZE + (width + 7) // 8 + valid * channels + 4


def parse(data: bytes) -> dict:
    """Token-packet parse + validation (transport.py:154-218, _check_seal 64-70)."""
    if len(data) < 4:
        raise OraclePacketError("packet shorter than its checksum")
    body = data[:-4]
    if _crc(body) != struct.unpack(">I", data[-4:])[0]:
        raise OraclePacketError("crc32 mismatch")
    if len(body) < 4:
        raise OraclePacketError("packet body too short")
    magic, version, kind = struct.unpack(">HBB", body[:4])
    if magic != MAGIC:
        raise OraclePacketError(f"bad magic 0x{magic:04X}")
    if version != VERSION:
        raise OraclePacketError(f"unsupported version {version}")
    if kind not in (KIND_I, KIND_P):
        raise OraclePacketError(f"unknown packet kind {kind}")
    if len(body) < HDR_SIZE:
        raise OraclePacketError("token packet header truncated")
    (_, _, _, gop_id, row, width, channels, scale, qmin, qrange) = \
        TOKEN_HDR.unpack(body[:HDR_SIZE])
    mlen = (width + 7) // 8
    if len(body) < HDR_SIZE + mlen:
        raise OraclePacketError("token packet mask truncated")
    bits = np.unpackbits(np.frombuffer(body[HDR_SIZE:HDR_SIZE + mlen], np.uint8))
    mask = bits[:width].astype(bool)
    payload = body[HDR_SIZE + mlen:]
    if len(payload) != int(mask.sum()) * channels:
        raise OraclePacketError(
            f"payload length {len(payload)} != popcount(mask)*C = {int(mask.sum()) * channels}")
    if qrange < 0.0:
        raise OraclePacketError("negative quantization range")
    return dict(kind=kind, gop_id=gop_id, row=row, width=width, channels=channels,
                scale=scale, qmin=qmin, qrange=qrange, mask=mask, payload=payload)


def reassemble(parsed: list, shape: tuple, stats: dict | None = None):
    """Zero-fill, first-wins reassembly (transport.py:274-305, 108-112)."""
    h, w, c = shape
    values = np.zeros((h, w, c), dtype=np.float64)
    mask = np.zeros((h, w), dtype=bool)
    seen = set()
    corrupt = 0
    for pk in parsed:
        if pk["row"] >= h:
            corrupt += 1
            continue
        if pk["row"] in seen:
            continue
        seen.add(pk["row"])
        rm = pk["mask"][:w]
        if rm.any():
            raw = np.frombuffer(pk["payload"], np.uint8).astype(np.float64)
            vecs = raw.reshape(int(pk["mask"].sum()), pk["channels"])
            values[pk["row"]][rm] = pk["qmin"] + vecs * (pk["qrange"] / 255.0)
        mask[pk["row"]] = rm
    if stats is not None:
        if corrupt:
            stats["corrupt"] = stats.get("corrupt", 0) + corrupt
        stats["rows_received"] = len(seen)
    return values, mask


# ---------------------------------------------------------------------------
# a16: decoder

def detokenize(values: np.ndarray, frame_shape: tuple) -> np.ndarray:
    """4-coefficient IDCT, crop, clip (codec.py:131-140); float64 result."""
    hb, wb, _ = values.shape
    coeffs = np.zeros((hb, wb, 3, BLOCK, BLOCK), dtype=np.float64)
    per = values.reshape(hb, wb, 3, 4)
    for k, (y, x) in enumerate(COEFF_POSITIONS):
        coeffs[..., y, x] = per[..., k]
    blocks = idctn2_8x8(coeffs)
    img = blocks.transpose(0, 3, 1, 4, 2).reshape(hb * BLOCK, wb * BLOCK, 3)
    h, w = frame_shape
    return np_clip01(img[:h, :w])


def decode(i_vals, p_vals, p_mask, frame_shape):
    """(I image, concealed P image) float32 (codec.py:160-186)."""
    if i_vals.shape != p_vals.shape:
        raise ValueError(f"token shape mismatch: {i_vals.shape} vs {p_vals.shape}")
    i_img = detokenize(i_vals, frame_shape)
    p_img = detokenize(p_vals, frame_shape)
    concealed = ~np.asarray(p_mask, bool)
    if concealed.any():
        pix = np.repeat(np.repeat(concealed, BLOCK, axis=0), BLOCK, axis=1)
        pix = pix[:frame_shape[0], :frame_shape[1]]
        p_img = np.where(pix[..., None], i_img, p_img)
    return i_img.astype(np.float32), p_img.astype(np.float32)


# ---------------------------------------------------------------------------
# a17/a18: upscale and blend

def _axis_coords(n_out: int, n_in: int, s: int):
    """codec.py:222-228."""
    coords = (np.arange(n_out) + 0.5) / s - 0.5
    coords = np.clip(coords, 0.0, n_in - 1.0)
    lo = np.floor(coords).astype(np.int64)
    hi = np.minimum(lo + 1, n_in - 1)
    return lo, hi, coords - lo


def bilinear(img: np.ndarray, s: int) -> np.ndarray:
    """Half-pixel-centre bilinear, float64 (codec.py:217-235)."""
    h, w = img.shape[:2]
    y0, y1, fy = _axis_coords(h * s, h, s)
    x0, x1, fx = _axis_coords(w * s, w, s)
    img = np.asarray(img, dtype=np.float64)
    gx = (1 - fx)[None, :, None]
    fxb = fx[None, :, None]
    top = img[y0][:, x0] * gx + img[y0][:, x1] * fxb
    bot = img[y1][:, x0] * gx + img[y1][:, x1] * fxb
    return top * (1 - fy)[:, None, None] + bot * fy[:, None, None]


def upscale(img: np.ndarray, s: int, crop: tuple | None = None) -> np.ndarray:
    """upscale_frame + optional crop (codec.py:238-245, 264-266), float32."""
    out = np_clip01(bilinear(img, s)).astype(np.float32)
    if crop is not None:
        out = out[:crop[0], :crop[1]]
    return out


def blend(prev9: list, curr9: list, n: int) -> list:
    """Replace frames 0..n-1 of curr by the Eq. 2 mix (codec.py:278-296)."""
    if n > GOP_SIZE:
        raise ValueError(f"blend width {n} exceeds GoP size {GOP_SIZE}")
    if n < 1:
        raise ValueError("blend width must be >= 1")
    out = list(curr9)
    for i in range(1, n + 1):
        alpha = (n - i) / n
        a = np.asarray(prev9[GOP_SIZE - n + i - 1], dtype=np.float64)
        b = np.asarray(curr9[i - 1], dtype=np.float64)
        out[i - 1] = np_clip01(alpha * a + (1.0 - alpha) * b).astype(np.float32)
    return out


# ---------------------------------------------------------------------------
# a19: metrics

def mse(a: np.ndarray, b: np.ndarray) -> float:
    d = np.asarray(a, np.float64) - np.asarray(b, np.float64)
    return float(np.mean(d * d))                   # video.py:265-270


def psnr_from_mse(err: float) -> float:
    import math
    if err <= 0.0:
        return PSNR_CAP_DB
    return min(PSNR_CAP_DB, 10.0 * math.log10(1.0 / err))   # video.py:279-282


def gop_psnr(ref9, test9) -> tuple[float, float]:
    errs = [mse(r, t) for r, t in zip(ref9, test9)]
    pooled = float(np.mean(errs))
    return psnr_from_mse(pooled), pooled           # video.py:318-322


def boundary_flicker(prev9, curr9, n: int, norm: str = "l1") -> float:
    """video.py:285-304 (frame i of the current GoP vs frame T-n+i of the previous)."""
    total = 0.0
    for i in range(1, n + 1):
        a = np.asarray(curr9[i - 1], np.float64)
        b = np.asarray(prev9[GOP_SIZE - n + i - 1], np.float64)
        if norm == "l1":
            total += float(np.mean(np.abs(a - b)))
        else:
            total += float(np.sqrt(np.mean((a - b) ** 2)))
    return total / n


def inter_frame_consistency(frames) -> float:
    """video.py:307-315."""
    frames = list(frames)
    if len(frames) < 2:
        return 0.0
    deltas = [float(np.mean(np.abs(np.asarray(frames[i + 1], np.float64)
                                   - np.asarray(frames[i], np.float64))))
              for i in range(len(frames) - 1)]
    return float(np.mean(deltas))


# ---------------------------------------------------------------------------
# raw-rgb24 boundary (the reference CLI's file formats, cli.py:52-61,181)

def frames_from_rgb24(raw: np.ndarray) -> np.ndarray:
    """load_raw_video's sample conversion (video.py:130-135): uint8 q ->
    float32(q) / 255 (a float32 array over a Python float stays float32)."""
    return np.asarray(raw, dtype=np.uint8).astype(np.float32) / 255.0


def rgb24_from_frames(frames: np.ndarray) -> np.ndarray:
    """write_raw_video's quantiser (video.py:139-143): the float32 product
    v * 255, rounded half to even, as uint8."""
    return np.rint(np.asarray(frames, dtype=np.float32) * 255.0).astype(np.uint8)


# ---------------------------------------------------------------------------
# full per-GoP pipeline (BASELINE.md §2 composition, session.py:134-170,323-348)

def pipeline_gop(frames9: np.ndarray, s: int, gop_id: int = 0, drop_rate: float = 0.0,
                 lost: set | None = None, prev_out: list | None = None,
                 blend_width: int = 2) -> dict:
    """down -> encode -> [sim -> mask -> apply] -> packetize -> parse ->
    reassemble -> decode -> up(crop) -> blend.  ``lost`` holds packet indices
    (I rows first, then P rows) removed between sender and receiver."""
    H, W = frames9.shape[1:3]
    work = frames9 if s == 1 else downscale(frames9, s)    # s == 1: direct tokenizer
    h, w = work.shape[1:3]
    i_vals, p_vals = encode(work)
    ht, wt = i_vals.shape[:2]
    full = np.ones((ht, wt), dtype=bool)
    p_mask = full.copy()
    drop = np.zeros((ht, wt), dtype=bool)
    sim0 = similarity(p_vals, i_vals)
    if drop_rate > 0.0:
        drop = top_k_mask(sim0, drop_count(drop_rate, sim0.size))
        p_vals, p_mask = apply_mask(p_vals, p_mask, drop)
    pk_i = packetize(KIND_I, gop_id, i_vals, full, s)
    pk_p = packetize(KIND_P, gop_id, p_vals, p_mask, s)
    wire = pk_i + pk_p
    recv = [d for j, d in enumerate(wire) if not lost or j not in lost]
    parsed = [parse(d) for d in recv]
    ri, mi = reassemble([q for q in parsed if q["kind"] == KIND_I], (ht, wt, CHANNELS))
    rp, mp = reassemble([q for q in parsed if q["kind"] == KIND_P], (ht, wt, CHANNELS))
    i_img, p_img = decode(ri, rp, mp, (h, w))
    if s == 1:
        up_i, up_p = i_img, p_img
    else:
        up_i = upscale(i_img, s, crop=(H, W))
        up_p = upscale(p_img, s, crop=(H, W))
    out = [up_i] + [up_p] * (GOP_SIZE - 1)
    if prev_out is not None:
        out = blend(prev_out, out, blend_width)
    return dict(work=work, i_vals=i_vals, p_vals=p_vals, p_mask=p_mask, drop=drop, sim=sim0,
                wire=wire, i_img=i_img, p_img=p_img, frames=out,
                rows_received=(len(ri_rows := [q for q in parsed if q["kind"] == KIND_I]),
                               len(parsed) - len(ri_rows)))
