"""ORACLE / TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference's residual enhancement layer
and its entropy coder (§8 f2):

* residual.py:62-127  compute / aggregate / sparsify_quantize / apply
* residual.py:143-217 encode_payload / decode_payload / fit_to_budget
* rangecoder.py:39-243 symbol mapping, adaptive order-0 model, carry-less
  32-bit range coder (integer only -> byte-exact by construction)

Reproduces the reference's arithmetic order (numpy reductions start at the
identity 0.0, float64 throughout) so results are bit-identical; pinned by
tests/test_residual_oracle.py against the live reference and the golden
fixtures in tests/golden/residual_golden.json.
"""

from __future__ import annotations

import numpy as np

DEFAULT_THETA = 0.02                 # residual.py:13
DEFAULT_QUANT_STEP = 1.0 / 127.0     # residual.py:14
GOP_SIZE = 9

EOS = 0                              # rangecoder.py:21-23
MAX_RUN = 255
ALPHABET = 510
_TOP = 1 << 24                       # rangecoder.py:25-29
_BOTTOM = 1 << 16
_MASK = (1 << 32) - 1
_MAX_TOTAL = _BOTTOM


class OracleStreamError(ValueError):
    """Mirror of rangecoder.CorruptStreamError (rangecoder.py:32-33)."""


# ---------------------------------------------------------------------------
# residual layer

def compute_residual(x9: np.ndarray, xhat9: np.ndarray) -> np.ndarray:
    """r(t) = x(t) - x_hat(t) in float64 (residual.py:62-73)."""
    return np.asarray(x9, np.float64) - np.asarray(xhat9, np.float64)


def aggregate(res: np.ndarray) -> np.ndarray:
    """Temporal mean: sequential sum from 0.0 over the window, / T (residual.py:76-83)."""
    res = np.asarray(res, np.float64)
    acc = 0.0 + res[0]
    for t in range(1, res.shape[0]):
        acc = acc + res[t]
    return acc / float(res.shape[0])


def sparsify(avg: np.ndarray, theta: float = DEFAULT_THETA,
             step: float = DEFAULT_QUANT_STEP) -> tuple:
    """(indices, qvalues) of the thresholded 8-bit residual (residual.py:86-105)."""
    flat = np.asarray(avg, np.float64).ravel()
    qv = np.clip(np.rint(flat / step), -127, 127).astype(np.int16)
    keep = (np.abs(flat) >= theta) & (qv != 0) & (np.abs(qv) * step >= theta)
    idx = np.flatnonzero(keep)
    return idx, qv[idx]


def dense_delta(indices, qvalues, step, dims) -> np.ndarray:
    out = np.zeros(int(np.prod(dims)), np.float64)
    out[indices] = np.asarray(qvalues).astype(np.float64) * step       # residual.py:56-59
    return out.reshape(dims)


def apply(frame: np.ndarray, delta: np.ndarray) -> np.ndarray:
    """clip(frame + delta) as float32 (residual.py:117-125)."""
    return np.clip(np.asarray(frame, np.float64) + delta, 0.0, 1.0).astype(np.float32)


# ---------------------------------------------------------------------------
# range coder

def value_symbol(v: int) -> int:
    return v + 383 if v < 0 else v + 382               # rangecoder.py:45-48


def scan_to_symbols(dense) -> list:
    """Zero runs (<= 255) + values + EOS (rangecoder.py:75-94)."""
    dense = np.asarray(dense)
    syms = []
    pos = 0
    for idx in np.flatnonzero(dense).tolist():
        gap = idx - pos
        while gap > MAX_RUN:
            syms.append(MAX_RUN)
            gap -= MAX_RUN
        if gap:
            syms.append(gap)
        syms.append(value_symbol(int(dense[idx])))
        pos = idx + 1
    syms.append(EOS)
    return syms


class _Model:
    """Adaptive order-0 counts, all ones initially, halved at total 2^16
    (rangecoder.py:122-149), kept as plain Python lists."""

    def __init__(self):
        self.counts = [1] * ALPHABET
        self.total = ALPHABET

    def bounds(self, sym):
        c = sum(self.counts[:sym])
        return c, c + self.counts[sym], self.total

    def find(self, target):
        c = 0
        for s, n in enumerate(self.counts):
            if c + n > target:
                return s, c
            c += n
        return ALPHABET - 1, c - self.counts[-1]

    def update(self, sym):
        self.counts[sym] += 1
        self.total += 1
        if self.total >= _MAX_TOTAL:
            self.counts = [(n + 1) // 2 for n in self.counts]
            self.total = sum(self.counts)


def encode_stream(symbols) -> bytes:
    """rangecoder.py:155-185 (integer arithmetic; `low` is not masked after
    `low += c*r`, exactly as in the reference)."""
    m = _Model()
    out = bytearray()
    low, rng = 0, _MASK
    for sym in symbols:
        c, d, total = m.bounds(int(sym))
        r = rng // total
        low += c * r
        rng = (d - c) * r
        while (low ^ (low + rng)) < _TOP or rng < _BOTTOM:
            if (low ^ (low + rng)) >= _TOP:
                rng = (_MASK + 1 - low) & (_BOTTOM - 1)
            out.append((low >> 24) & 0xFF)
            low = (low << 8) & _MASK
            rng <<= 8
        m.update(int(sym))
    for _ in range(4):
        out.append((low >> 24) & 0xFF)
        low = (low << 8) & _MASK
    return bytes(out)


def decode_stream(data: bytes, max_symbols: int = 1 << 24) -> list:
    """rangecoder.py:188-235."""
    m = _Model()
    pos = 0

    def nb():
        nonlocal pos
        if pos >= len(data):
            raise OracleStreamError(f"compressed stream truncated at byte {pos} of {len(data)}")
        b = data[pos]
        pos += 1
        return b

    state = 0
    for _ in range(4):
        state = (state << 8) | nb()
    low, rng = 0, _MASK
    syms = []
    while True:
        total = m.total
        r = rng // total
        val = (state - low) // r
        if val >= total:
            val = total - 1
        sym, c = m.find(val)
        syms.append(sym)
        d = c + m.counts[sym]
        low += c * r
        rng = (d - c) * r
        while (low ^ (low + rng)) < _TOP or rng < _BOTTOM:
            if (low ^ (low + rng)) >= _TOP:
                rng = (_MASK + 1 - low) & (_BOTTOM - 1)
            state = ((state << 8) | nb()) & _MASK
            low = (low << 8) & _MASK
            rng <<= 8
        m.update(sym)
        if sym == EOS:
            return syms
        if len(syms) >= max_symbols:
            raise OracleStreamError("symbol budget exceeded before EOS")


def symbols_to_scan(symbols, length: int) -> np.ndarray:
    """rangecoder.py:97-116."""
    out = np.zeros(length, np.int16)
    pos = 0
    for i, s in enumerate(symbols):
        if s == EOS:
            if i != len(symbols) - 1:
                raise OracleStreamError(f"EOS at position {i} before end of stream")
            return out
        if 1 <= s <= MAX_RUN:
            pos += s
            if pos > length:
                raise OracleStreamError(f"zero run overruns scan length {length}")
        else:
            if pos >= length:
                raise OracleStreamError(f"value overruns scan length {length}")
            out[pos] = s - 383 if s <= 382 else s - 382
            pos += 1
    raise OracleStreamError("symbol stream missing EOS")


def encode_scan(dense) -> bytes:
    return encode_stream(scan_to_symbols(dense))


def decode_scan(data: bytes, length: int) -> np.ndarray:
    return symbols_to_scan(decode_stream(data), length)


# ---------------------------------------------------------------------------
# budget fitting (residual.py:159-217)

def fit_to_budget(avg, budget, step=DEFAULT_QUANT_STEP, theta_floor=DEFAULT_THETA,
                  max_trials=6):
    """Returns (indices, qvalues, payload, theta) or (None, None, b"", theta)."""
    if budget <= 0:
        return None, None, b"", float("inf")
    avg = np.asarray(avg, np.float64)
    idx, qv = sparsify(avg, theta_floor, step)
    if idx.size == 0:
        return None, None, b"", theta_floor
    mags = np.abs(avg.ravel()[idx])
    order = np.argsort(-mags, kind="stable")
    lookup = np.zeros(avg.size, np.int16)
    lookup[idx] = qv
    full_k = idx.size

    def dense_of(ind):
        d = np.zeros(avg.size, np.int16)
        d[ind] = lookup[ind]
        return d

    def build(k):
        if k >= full_k:
            return idx, theta_floor
        chosen = np.sort(idx[order[:k]])
        return chosen, float(np.min(np.abs(lookup[chosen])) * step)

    k = full_k if full_k <= 2 * budget else int(budget)
    best = None
    for _ in range(max_trials):
        k = max(1, min(k, full_k))
        chosen, theta = build(k)
        payload = encode_scan(dense_of(chosen))
        if len(payload) <= budget:
            best = (chosen, lookup[chosen], payload, theta)
            if k >= full_k or len(payload) >= 0.80 * budget:
                return best
            grown = int(k * budget / max(len(payload), 1) * 0.95)
            if grown <= k:
                return best
            k = grown
        else:
            shrunk = int(k * budget / len(payload) * 0.92)
            if shrunk < 1 or (best is not None and shrunk <= best[0].size):
                break
            k = shrunk
    if best is not None:
        return best
    return None, None, b"", float("inf")
