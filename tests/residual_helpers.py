"""Input regeneration for tests/golden/residual_golden.json (mirrors
tests/golden/make_residual_golden.py)."""

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden" / "residual_golden.json"


def golden():
    return json.loads(GOLDEN.read_text())


def avg_input(seed, shape, scale):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal(tuple(shape)) * scale
    a[rng.random(tuple(shape)) < 0.3] = 0.0
    return a


def symbol_stream(seed, n):
    rng = np.random.default_rng(seed)
    return [int(s) for s in rng.integers(1, 510, size=n)] + [0]
