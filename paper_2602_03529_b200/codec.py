"""Tokenizer, scaling and boundary blending -- drop-in for ``semstream.codec``
(reference pkg/src/semstream/codec.py), executed by the sm_100a kernels.

Same names, signatures, dataclasses, validation and error types as the
reference; every numeric result is produced on the GPU through the C ABI
(``include/semstream_b200.h``) and is bit-identical to the reference's numpy /
scipy computation.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _dev, _lib
from .video import GOP_SIZE, Frame, GoP

BLOCK = 8                                              # codec.py:20
COEFF_POSITIONS = ((0, 0), (0, 1), (1, 0), (2, 0))     # codec.py:22
COEFFS_PER_CHANNEL = len(COEFF_POSITIONS)


@dataclass(frozen=True)
class CodecConfig:
    """codec.py:26-46 (factors fixed at 8, scale in {2,3}, blend width 1..8)."""

    spatial_factor: int = 8
    temporal_factor: int = 8
    channels: int = 3 * COEFFS_PER_CHANNEL
    scale: int = 3
    blend_width: int = 2

    def __post_init__(self):
        if self.spatial_factor != 8 or self.temporal_factor != 8:
            raise ValueError("spatial and temporal compression factors are fixed at 8")
        if self.scale not in (2, 3):
            raise ValueError(f"scale must be 2 or 3, got {self.scale}")
        if not 1 <= self.blend_width <= 8:
            raise ValueError(f"blend width must be in [1, 8], got {self.blend_width}")
        if self.channels != 3 * COEFFS_PER_CHANNEL:
            raise ValueError(f"reference tokenizer emits {3 * COEFFS_PER_CHANNEL} channels, "
                             f"got {self.channels}")


@dataclass(frozen=True)
class TokenMatrix:
    """H' x W' x C float64 latent grid with validity mask (codec.py:49-91)."""

    kind: str
    values: np.ndarray
    mask: np.ndarray
    gop_id: int = 0
    frame_shape: tuple | None = None

    def __post_init__(self):
        if self.kind not in ("I", "P"):
            raise ValueError(f"token matrix kind must be 'I' or 'P', got {self.kind!r}")
        values = np.asarray(self.values, dtype=np.float64)
        mask = np.asarray(self.mask, dtype=bool)
        if values.ndim != 3:
            raise ValueError(f"token values must be (H', W', C), got {values.shape}")
        if mask.shape != values.shape[:2]:
            raise ValueError(f"mask shape {mask.shape} does not match {values.shape[:2]}")
        if not np.isfinite(values).all():
            raise ValueError("token values must be finite")
        if np.any(values[~mask] != 0.0):
            raise ValueError("masked-out token positions must be exactly zero")
        object.__setattr__(self, "values", values)
        object.__setattr__(self, "mask", mask)
        if self.frame_shape is not None:
            object.__setattr__(self, "frame_shape", tuple(self.frame_shape))

    @property
    def height_tokens(self) -> int:
        return self.values.shape[0]

    @property
    def width_tokens(self) -> int:
        return self.values.shape[1]

    @property
    def channels(self) -> int:
        return self.values.shape[2]


def token_grid_shape(height: int, width: int) -> tuple:
    """(H', W') = ceil(dims / 8) (codec.py:94-96)."""
    return (-(-height // BLOCK), -(-width // BLOCK))


# ---------------------------------------------------------------------------
# tokenizer

def encode_gop(gop: GoP, cfg: CodecConfig) -> tuple:
    """I tokens from frame 0, P tokens from the mean of frames 1..8
    (codec.py:143-157), computed by ``sst_encode`` (s = 1)."""
    if len(gop.frames) != GOP_SIZE:
        raise ValueError(f"GoP must hold {GOP_SIZE} frames")
    h, w = gop.height, gop.width
    ht, wt = token_grid_shape(h, w)
    frames = _dev.h2d(gop.stacked(), np.float32)
    tok = _dev.empty((1, 2, ht, wt, 3 * COEFFS_PER_CHANNEL), torch.float64)
    _lib.call("sst_encode", _dev.ptr(frames), 1, h, w, 1, _dev.ptr(tok), None, _dev.stream())
    t = _dev.d2h(tok)[0]
    full = np.ones((ht, wt), dtype=bool)
    i_tokens = TokenMatrix("I", t[0], full, gop_id=gop.gop_id, frame_shape=(h, w))
    p_tokens = TokenMatrix("P", t[1], full.copy(), gop_id=gop.gop_id, frame_shape=(h, w))
    return i_tokens, p_tokens


def decode_gop(i_tokens: TokenMatrix, p_tokens: TokenMatrix, cfg: CodecConfig) -> GoP:
    """IDCT + temporal-reference concealment (codec.py:160-186) via ``sst_decode``.
    Frames 1..8 share one buffer, as in the reference."""
    if i_tokens.values.shape != p_tokens.values.shape:
        raise ValueError(
            f"token shape mismatch: {i_tokens.values.shape} vs {p_tokens.values.shape}")
    ht, wt, c = i_tokens.values.shape
    if c != 3 * COEFFS_PER_CHANNEL:
        raise ValueError(f"decoder expects {3 * COEFFS_PER_CHANNEL} channels, got {c}")
    shape = i_tokens.frame_shape or (ht * BLOCK, wt * BLOCK)
    h, w = min(shape[0], ht * BLOCK), min(shape[1], wt * BLOCK)   # numpy slice semantics
    iv = _dev.h2d(i_tokens.values, np.float64)
    pv = _dev.h2d(p_tokens.values, np.float64)
    pm = _dev.h2d(p_tokens.mask, np.uint8)
    out = _dev.empty((1, 2, h, w, 3), torch.float32)
    _lib.call("sst_decode", _dev.ptr(iv), _dev.ptr(pv), 0, _dev.ptr(pm), 1, ht, wt, h, w,
              _dev.ptr(out), _dev.stream())
    imgs = _dev.d2h(out)[0]
    frames = [Frame(imgs[0], timestamp_index=0)]
    p_frame = imgs[1]
    for t in range(1, GOP_SIZE):
        frames.append(Frame(p_frame, timestamp_index=t))
    return GoP(gop_id=i_tokens.gop_id, frames=tuple(frames))


def apply_token_mask(matrix: TokenMatrix, drop_mask: np.ndarray) -> TokenMatrix:
    """Zero and invalidate dropped positions (codec.py:189-196)."""
    drop = np.asarray(drop_mask, dtype=bool)
    if drop.shape != matrix.mask.shape:
        raise ValueError(f"drop mask shape {drop.shape} != {matrix.mask.shape}")
    vals = _dev.h2d(matrix.values, np.float64)
    mask = _dev.h2d(matrix.mask, np.uint8)
    dr = _dev.h2d(drop, np.uint8)
    n = matrix.mask.size
    _lib.call("sst_apply_mask", _dev.ptr(vals), _dev.ptr(mask), _dev.ptr(dr), n,
              matrix.channels, _dev.stream())
    return replace(matrix, values=_dev.d2h(vals), mask=_dev.d2h(mask).astype(bool))


# ---------------------------------------------------------------------------
# resolution scaling

def _check_scale(s: int) -> None:
    if s not in (2, 3):
        raise ValueError(f"scale factor must be 2 or 3, got {s}")


def _downscale_stack(stack: np.ndarray, s: int) -> np.ndarray:
    n, h, w = stack.shape[:3]
    src = _dev.h2d(stack, np.float32)
    out = _dev.empty((n, -(-h // s), -(-w // s), 3), torch.float32)
    _lib.call("sst_downscale", _dev.ptr(src), n, h, w, s, _dev.ptr(out), _dev.stream())
    return _dev.d2h(out)


def downscale_frame(frame: Frame, s: int) -> Frame:
    """s x s box mean with edge replication (codec.py:202-214)."""
    _check_scale(s)
    out = _downscale_stack(frame.samples[None], s)[0]
    return Frame(out, timestamp_index=frame.timestamp_index)


def bilinear_upscale(img: np.ndarray, s: int) -> np.ndarray:
    """Half-pixel-centre bilinear x s, float64, unclipped (codec.py:217-235)."""
    arr = np.asarray(img, dtype=np.float64)
    if arr.ndim != 3 or arr.shape[2] != 3:
        raise ValueError(f"expected an (h, w, 3) image, got {arr.shape}")
    h, w = arr.shape[:2]
    src = _dev.h2d(arr)
    out = _dev.empty((1, h * s, w * s, 3), torch.float64)
    _lib.call("sst_bilinear_f64", _dev.ptr(src), 1, h, w, s, _dev.ptr(out), _dev.stream())
    return _dev.d2h(out)[0]


def _upscale_stack(stack: np.ndarray, s: int, crop) -> np.ndarray:
    n, h, w = stack.shape[:3]
    ch, cw = h * s, w * s
    if crop is not None:
        ch, cw = min(crop[0], ch), min(crop[1], cw)
    src = _dev.h2d(stack, np.float32)
    out = _dev.empty((n, ch, cw, 3), torch.float32)
    _lib.call("sst_upscale", _dev.ptr(src), n, h, w, s, ch, cw, _dev.ptr(out), _dev.stream())
    return _dev.d2h(out)


def _clip_cast(arr: np.ndarray) -> np.ndarray:
    x = _dev.h2d(np.asarray(arr), np.float64)
    out = _dev.empty(x.shape, torch.float32)
    _lib.call("sst_clip_cast", _dev.ptr(x), x.numel(), _dev.ptr(out), _dev.stream())
    return _dev.d2h(out)


def upscale_frame(frame: Frame, s: int, upscaler=None) -> Frame:
    """Upscale by s with a pluggable upscaler (codec.py:238-245)."""
    _check_scale(s)
    if upscaler is not None:
        out = _clip_cast(upscaler(frame.samples, s))
    else:
        out = _upscale_stack(frame.samples[None], s, None)[0]
    return Frame(out, timestamp_index=frame.timestamp_index)


def scale_gop(gop: GoP, s: int, direction: str, upscaler=None, crop: tuple | None = None) -> GoP:
    """Scale every frame of a GoP (codec.py:248-272); shared sample buffers are
    upscaled once."""
    if direction == "down":
        _check_scale(s)
        out = _downscale_stack(gop.stacked(), s)
        frames = [Frame(out[i], timestamp_index=f.timestamp_index)
                  for i, f in enumerate(gop.frames)]
        return GoP(gop_id=gop.gop_id, frames=tuple(frames), scale=s)
    if direction == "up":
        _check_scale(s)
        uniq: dict = {}
        for f in gop.frames:
            uniq.setdefault(id(f.samples), f)
        keys = list(uniq)
        if upscaler is None:
            outs = _upscale_stack(np.stack([uniq[k].samples for k in keys]), s, crop)
            cache = {k: outs[j] for j, k in enumerate(keys)}
        else:
            cache = {}
            for k in keys:
                o = _clip_cast(upscaler(uniq[k].samples, s))
                if crop is not None:
                    o = o[:crop[0], :crop[1]]
                cache[k] = o
        frames = [Frame(cache[id(f.samples)], timestamp_index=f.timestamp_index)
                  for f in gop.frames]
        return GoP(gop_id=gop.gop_id, frames=tuple(frames), scale=1)
    raise ValueError(f"direction must be 'down' or 'up', got {direction!r}")


# ---------------------------------------------------------------------------
# boundary blending

def blend_boundary(prev_recon: GoP, curr_recon: GoP, n: int) -> GoP:
    """Eq. 2 boundary blend of the first n frames (codec.py:278-296)."""
    if n > GOP_SIZE:
        raise ValueError(f"blend width {n} exceeds GoP size {GOP_SIZE}")
    if n < 1:
        raise ValueError("blend width must be >= 1")
    if (prev_recon.height, prev_recon.width) != (curr_recon.height, curr_recon.width):
        raise ValueError("GoP dimension mismatch")
    H, W = curr_recon.height, curr_recon.width
    prev = _dev.h2d(prev_recon.stacked(), np.float32)
    curr = _dev.h2d(curr_recon.stacked(), np.float32)
    _lib.call("sst_blend", _dev.ptr(prev), _dev.ptr(curr), 1, H, W, n, _dev.ptr(curr),
              _dev.stream())
    mixed = _dev.d2h(curr[:n])
    frames = list(curr_recon.frames)
    for i in range(n):
        frames[i] = Frame(mixed[i], timestamp_index=curr_recon.frames[i].timestamp_index)
    return GoP(gop_id=curr_recon.gop_id, frames=tuple(frames), scale=curr_recon.scale)
