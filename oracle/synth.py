"""ORACLE / TEST INFRASTRUCTURE ONLY.

Restatement of the reference's seeded synthetic clips
(pkg/src/semstream/synth.py:56-171) so that parity tests and the CPU baseline
can regenerate byte-identical input frames without /root/reference.  Random
draws are made in exactly the reference's order.
"""

from __future__ import annotations

import numpy as np

from .semstream_oracle import GOP_SIZE, bilinear


def gradient(width: int, height: int, phase: float = 0.0) -> np.ndarray:
    """synth.py:56-62."""
    x = np.linspace(0.0, 1.0, width)[None, :]
    y = np.linspace(0.0, 1.0, height)[:, None]
    r = np.broadcast_to(0.25 + 0.5 * x, (height, width))
    g = np.broadcast_to(0.25 + 0.5 * y, (height, width))
    b = np.full((height, width), 0.4 + 0.2 * np.sin(phase))
    return np.clip(np.stack([r, g, b], axis=2), 0.0, 1.0)


class Clip:
    """Frame source addressable by frame / GoP index (synth.py:12-53)."""

    def __init__(self, name, width, height, frame_count, seed=0, **kw):
        if frame_count <= 0:
            raise ValueError("frame_count must be positive")
        self.name, self.width, self.height = name, width, height
        self.frame_count, self.seed = frame_count, seed
        w, h = width, height
        if name == "static-gradient":                      # synth.py:65-73
            self._img = gradient(w, h)
        elif name == "moving-square":                      # synth.py:76-97
            self._bg = gradient(w, h)
            self.side = max(8, int(min(w, h) * kw.get("square_frac", 0.25)))
            self.speed = kw.get("speed", 4)
            rng = np.random.default_rng(seed)
            tex = rng.random((self.side // 4 + 1, self.side // 4 + 1, 3))
            self._tex = np.repeat(np.repeat(tex, 4, axis=0), 4, axis=1)[:self.side, :self.side]
        elif name == "noise-field":                        # synth.py:100-111
            self._bg = gradient(w, h)
            self.amp = kw.get("amplitude", 0.5)
        elif name == "noisy-motion":                       # synth.py:114-136
            rng = np.random.default_rng(seed)
            base = gradient(w, h)
            self._bg = np.clip(base + kw.get("static_noise", 0.3) * (rng.random((h, w, 3)) - 0.5),
                               0.0, 1.0)
            self.frame_noise = kw.get("frame_noise", 0.15)
            self.side = max(8, min(w, h) // 4)
            self.speed = kw.get("speed", 6)
        elif name == "static-detail":                      # synth.py:139-162
            scale = kw.get("scale", 2)
            wh, ww = -(-h // scale), -(-w // scale)
            rng = np.random.default_rng(seed)
            img = gradient(ww, wh)
            for _ in range(40):
                rw = int(rng.integers(4, ww // 4))
                rh = int(rng.integers(4, wh // 4))
                x0 = int(rng.integers(0, ww - rw))
                y0 = int(rng.integers(0, wh - rh))
                img[y0:y0 + rh, x0:x0 + rw] = rng.random(3)
            self._img = np.clip(bilinear(img, scale)[:h, :w], 0.0, 1.0)
        else:
            raise ValueError(f"unknown synthetic clip {name!r}")

    @property
    def gop_count(self) -> int:
        return -(-self.frame_count // GOP_SIZE)

    def frame_array(self, i: int) -> np.ndarray:
        n = self.name
        if n in ("static-gradient", "static-detail"):
            return self._img
        if n == "moving-square":
            img = self._bg.copy()
            x = (self.speed * i) % max(self.width - self.side, 1)
            y = (self.speed * i // 2) % max(self.height - self.side, 1)
            img[y:y + self.side, x:x + self.side] = self._tex
            return img
        if n == "noise-field":
            rng = np.random.default_rng((self.seed, i))
            noise = rng.random((self.height, self.width, 3)) - 0.5
            return np.clip(self._bg + self.amp * noise, 0.0, 1.0)
        # noisy-motion
        img = self._bg.copy()
        x = (self.speed * i) % max(self.width - self.side, 1)
        y = (self.speed * i // 2) % max(self.height - self.side, 1)
        img[y:y + self.side, x:x + self.side] = 1.0 - img[y:y + self.side, x:x + self.side]
        rng = np.random.default_rng((self.seed, 7919, i))
        noise = rng.random((self.height, self.width, 3)) - 0.5
        return np.clip(img + self.frame_noise * noise, 0.0, 1.0)

    def frame(self, i: int) -> np.ndarray:
        """float32 frame with tail padding (synth.py:35-37)."""
        return self.frame_array(min(i, self.frame_count - 1)).astype(np.float32)

    def gop(self, k: int) -> np.ndarray:
        """(9, H, W, 3) float32 (synth.py:39-50)."""
        if not 0 <= k < self.gop_count:
            raise ValueError(f"gop index {k} out of range [0, {self.gop_count})")
        return np.stack([self.frame(k * GOP_SIZE + t) for t in range(GOP_SIZE)])


def make_clip(name: str, width: int, height: int, frame_count: int, seed: int = 0) -> Clip:
    """synth.py:174-180."""
    return Clip(name, width, height, frame_count, seed)
