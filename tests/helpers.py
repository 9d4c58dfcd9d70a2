"""Shared test helpers: golden fixtures, input regeneration, digests, and
the reference suite's frame fixtures (pkg/tests/conftest.py:7-24)."""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np

from oracle import semstream_oracle as O
from oracle.synth import make_clip

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden.json"


def digest(a) -> str:
    if isinstance(a, (bytes, bytearray)):
        return hashlib.sha256(bytes(a)).hexdigest()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def wire_digest(wire) -> str:
    return digest(b"".join(len(d).to_bytes(4, "big") + d for d in wire))


def golden():
    return json.loads(GOLDEN.read_text())


def golden_cases(max_pixels: int | None = None):
    out = []
    for c in golden()["cases"]:
        cc = c["case"]
        if max_pixels is None or cc["W"] * cc["H"] <= max_pixels:
            out.append(c)
    return out


def case_clip(cc: dict):
    return make_clip(cc["clip"], cc["W"], cc["H"], cc["frames"], seed=cc["seed"])


def oracle_case(c: dict):
    """Run the oracle over a golden case; yields (gop_record, oracle_result)."""
    cc = c["case"]
    clip = case_clip(cc)
    prev = None
    for k, rec in enumerate(c["gops"]):
        frames = clip.gop(k)
        res = O.pipeline_gop(frames, rec["scale"], gop_id=k, drop_rate=cc["drop"],
                             lost=set(rec["lost"]), prev_out=prev)
        prev = res["frames"]
        yield rec, frames, res


# pkg/tests/conftest.py:7-24 fixtures, as plain arrays
def random_frame(rng, h=16, w=16, dyadic=False):
    arr = rng.random((h, w, 3))
    if dyadic:
        arr = np.floor(arr * 256.0) / 256.0
    return arr.astype(np.float32)


def random_gop(rng, h=16, w=16, dyadic=False):
    return np.stack([random_frame(rng, h, w, dyadic) for _ in range(9)])
