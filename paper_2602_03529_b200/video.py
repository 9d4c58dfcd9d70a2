"""Data model and quality metrics of the codec path -- drop-in for
``semstream.video`` (reference pkg/src/semstream/video.py).

``Frame`` / ``GoP`` keep the reference's value semantics and validation
(video.py:20-86).  The pixel metrics run on the GPU (``sst_mse`` and device
reductions); raw-video / y4m file I/O is outside the codec hot path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib

GOP_SIZE = 9          # video.py:12
PSNR_CAP_DB = 99.0    # video.py:13


@dataclass(frozen=True)
class Frame:
    """One RGB frame; samples are (h, w, 3) float32 in [0, 1] (video.py:20-54)."""

    samples: np.ndarray
    timestamp_index: int = 0

    def __post_init__(self):
        arr = np.asarray(self.samples, dtype=np.float32)
        if arr.ndim != 3 or arr.shape[2] != 3:
            raise ValueError(f"frame samples must be (h, w, 3), got {arr.shape}")
        if arr.shape[0] <= 0 or arr.shape[1] <= 0:
            raise ValueError("frame dimensions must be positive")
        if not np.isfinite(arr).all():
            raise ValueError("frame samples must be finite")
        lo, hi = float(arr.min()), float(arr.max())
        if lo < 0.0 or hi > 1.0:
            raise ValueError(f"frame samples outside [0, 1]: min={lo}, max={hi}")
        object.__setattr__(self, "samples", arr)

    @property
    def height(self) -> int:
        return self.samples.shape[0]

    @property
    def width(self) -> int:
        return self.samples.shape[1]

    @property
    def channels(self) -> int:
        return 3


@dataclass(frozen=True)
class GoP:
    """One I frame followed by eight P frames (video.py:57-86)."""

    gop_id: int
    frames: tuple
    scale: int = 1

    def __post_init__(self):
        frames = tuple(self.frames)
        if len(frames) != GOP_SIZE:
            raise ValueError(f"a GoP holds exactly {GOP_SIZE} frames, got {len(frames)}")
        dims = {(f.height, f.width) for f in frames}
        if len(dims) != 1:
            raise ValueError(f"mixed frame dimensions in GoP: {sorted(dims)}")
        if self.scale not in (1, 2, 3):
            raise ValueError(f"scale must be 1, 2 or 3, got {self.scale}")
        object.__setattr__(self, "frames", frames)

    @property
    def height(self) -> int:
        return self.frames[0].height

    @property
    def width(self) -> int:
        return self.frames[0].width

    def stacked(self) -> np.ndarray:
        return np.stack([f.samples for f in self.frames])


@dataclass(frozen=True)
class QualityReport:
    psnr_db: float
    mse: float
    boundary_flicker: float
    consistency_delta: float

    def __post_init__(self):
        for name in ("psnr_db", "mse", "boundary_flicker", "consistency_delta"):
            if getattr(self, name) < 0.0:
                raise ValueError(f"{name} must be non-negative")


def segment_gops(frames, start_gop_id: int = 0) -> list:
    """9-frame GoPs with last-frame tail padding (video.py:236-251)."""
    frames = list(frames)
    if not frames:
        raise ValueError("cannot segment an empty frame sequence")
    dims = {(f.height, f.width) for f in frames}
    if len(dims) != 1:
        raise ValueError(f"mixed frame dimensions: {sorted(dims)}")
    gops = []
    for k in range(0, len(frames), GOP_SIZE):
        chunk = frames[k:k + GOP_SIZE]
        while len(chunk) < GOP_SIZE:
            chunk.append(chunk[-1])
        gops.append(GoP(gop_id=start_gop_id + k // GOP_SIZE, frames=tuple(chunk)))
    return gops


def concat_gops(gops, frame_count: int | None = None) -> list:
    """Inverse of segment_gops (video.py:254-259)."""
    frames = [f for g in gops for f in g.frames]
    if frame_count is not None:
        frames = frames[:frame_count]
    return frames


# ---------------------------------------------------------------------------
# metrics (device reductions)

def _mean_diff(refs, tests, mode: int = 0) -> np.ndarray:
    """np.mean of the float64 per-pixel (a-b)^2 (mode 0) or |a-b| (mode 1) of
    each frame pair, on the GPU in numpy's pairwise summation order
    (csrc/metrics.cu): bit-identical to the reference's metric arithmetic."""
    refs = [np.asarray(getattr(r, "samples", r)) for r in refs]
    tests = [np.asarray(getattr(t, "samples", t)) for t in tests]
    for r, t in zip(refs, tests):
        if r.shape != t.shape:
            raise ValueError(f"dimension mismatch: {r.shape} vs {t.shape}")
    if not refs:
        return np.zeros(0)
    a = _dev.h2d(np.stack(refs), np.float32)
    b = _dev.h2d(np.stack(tests), np.float32)
    out = _dev.empty((len(refs),), torch.float64)
    elems = int(np.prod(refs[0].shape))
    _lib.call("sst_mean_diff", _dev.ptr(a), _dev.ptr(b), len(refs), elems, mode, _dev.ptr(out),
              _dev.stream())
    return _dev.d2h(out)


def _mse_many(refs, tests) -> np.ndarray:
    return _mean_diff(refs, tests, 0)


def gop_psnr_device(reference: torch.Tensor, test: torch.Tensor) -> tuple:
    """gop_psnr (video.py:318-322) of device GoPs: float32 [9, H, W, 3] CUDA
    tensors, reduced in place on the GPU (no host copy of the frames)."""
    if reference.shape != test.shape or reference.dim() != 4:
        raise ValueError(f"dimension mismatch: {tuple(reference.shape)} vs {tuple(test.shape)}")
    if reference.dtype != torch.float32 or test.dtype != torch.float32:
        raise ValueError("frames must be float32")
    a, b = reference.contiguous(), test.contiguous()
    out = torch.empty((a.shape[0],), dtype=torch.float64, device=a.device)
    _lib.call("sst_mean_diff", a.data_ptr(), b.data_ptr(), a.shape[0], a[0].numel(), 0,
              out.data_ptr(), _dev.stream())
    pooled = float(np.mean(_dev.d2h(out)))
    return psnr_from_mse(pooled), pooled


def mse(reference: Frame, test: Frame) -> float:
    """video.py:265-270."""
    return float(_mse_many([reference], [test])[0])


def psnr_from_mse(err: float) -> float:
    if err <= 0.0:
        return PSNR_CAP_DB
    return min(PSNR_CAP_DB, 10.0 * math.log10(1.0 / err))    # video.py:279-282


def psnr(reference: Frame, test: Frame) -> float:
    return psnr_from_mse(mse(reference, test))


def gop_psnr(reference: GoP, test: GoP) -> tuple:
    """(psnr_db, mse) pooled over the 9 frames (video.py:318-322)."""
    errs = _mse_many(reference.frames, test.frames)
    pooled = float(np.mean(errs))
    return psnr_from_mse(pooled), pooled


def boundary_flicker(prev_gop_recon: GoP, curr_gop_recon: GoP, n: int, norm: str = "l1") -> float:
    """Mean |curr[i] - prev[T-n+i]| over the n boundary frames (video.py:285-304)."""
    if not 1 <= n <= GOP_SIZE:
        raise ValueError(f"blend width n must be in [1, {GOP_SIZE}], got {n}")
    if (prev_gop_recon.height, prev_gop_recon.width) != (curr_gop_recon.height, curr_gop_recon.width):
        raise ValueError("GoP dimension mismatch")
    if norm not in ("l1", "l2"):
        raise ValueError(f"unknown norm {norm!r}")
    per = _mean_diff([curr_gop_recon.frames[i - 1] for i in range(1, n + 1)],
                     [prev_gop_recon.frames[GOP_SIZE - n + i - 1] for i in range(1, n + 1)],
                     1 if norm == "l1" else 0)
    total = 0.0
    for v in per:                                    # video.py:294-303, in order
        total += float(v) if norm == "l1" else float(np.sqrt(v))
    return total / n


def inter_frame_consistency(frames) -> float:
    """Mean absolute inter-frame pixel difference (video.py:307-315)."""
    frames = list(frames)
    if len(frames) < 2:
        return 0.0
    deltas = _mean_diff(frames[1:], frames[:-1], 1)
    return float(np.mean([float(d) for d in deltas]))


def quality_report(reference: GoP, test: GoP, prev_recon: GoP | None = None,
                   blend_width: int = 2) -> QualityReport:
    psnr_db, pooled = gop_psnr(reference, test)
    flicker = 0.0
    if prev_recon is not None:
        flicker = boundary_flicker(prev_recon, test, blend_width)
    return QualityReport(psnr_db=psnr_db, mse=pooled, boundary_flicker=flicker,
                         consistency_delta=inter_frame_consistency(test.frames))
