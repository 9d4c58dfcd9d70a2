"""GPU: residual enhancement layer and range coder against
the live-reference fixtures, the oracle, and the reference suite's own
test_rangecoder.py / test_residual.py cases."""

import math

import numpy as np
import pytest

from helpers import digest
from oracle import residual_oracle as R
from oracle import semstream_oracle as O
from oracle.synth import make_clip
from paper_2602_03529_b200 import codec as C, rangecoder as RC, residual as RS, video as V
from residual_helpers import avg_input, golden, symbol_stream

pytestmark = pytest.mark.gpu
G = golden()


@pytest.mark.parametrize("c", G["cases"], ids=[str(c["seed"]) for c in G["cases"]])
def test_sparsify_encode_fit_match_reference(c):
    avg = avg_input(c["seed"], c["shape"], c["scale"])
    sr = RS.sparsify_quantize(avg)
    assert digest(sr.indices) == c["indices"] and digest(sr.qvalues) == c["qvalues"]
    payload = RS.encode_payload(sr)
    assert digest(payload) == c["payload"]
    back = RS.decode_payload(payload, avg.shape, sr.theta, sr.quant_step, 9)
    assert np.array_equal(back.indices, sr.indices) and np.array_equal(back.qvalues, sr.qvalues)
    for f in c["fits"]:
        got, pay, theta = RS.fit_to_budget(avg, f["budget"])
        assert (got is None) == f["none"]
        assert digest(pay) == f["payload"] and theta == f["theta"]
        if got is not None:
            assert digest(got.indices) == f["indices"] and digest(got.qvalues) == f["qvalues"]


@pytest.mark.parametrize("s", G["streams"], ids=[str(s["seed"]) for s in G["streams"]])
def test_symbol_streams_match_reference(s):
    syms = symbol_stream(s["seed"], s["n"])
    data = RC.encode_stream(syms)
    assert digest(data) == s["data"]
    assert RC.decode_stream(data) == syms


def test_session_residual_matches_reference():
    s = G["session"]
    src = make_clip(s["clip"], s["W"], s["H"], 9, seed=s["seed"]).gop(0)
    g = V.GoP(0, tuple(V.Frame(f, timestamp_index=t) for t, f in enumerate(src)))
    work = C.scale_gop(g, s["scale"], "down")
    cfg = C.CodecConfig()
    rec = C.decode_gop(*C.encode_gop(work, cfg), cfg)
    res = RS.compute_residual(work, rec)
    assert digest(res) == s["residual"]
    avg = RS.aggregate_residual(res)
    assert digest(avg) == s["avg"]
    sr, payload, theta = RS.fit_to_budget(avg, s["budget"])
    assert digest(sr.indices) == s["indices"] and digest(payload) == s["payload"]
    assert theta == s["theta"]
    applied = RS.apply_residual(rec, sr)
    assert digest(np.stack([f.samples for f in applied.frames])) == s["applied"]
    assert applied.frames[1].samples is applied.frames[8].samples


def test_batched_coding_many_streams(rng):
    scans = []
    for i in range(12):
        n = 5000
        d = np.where(rng.random(n) < [0.001, 0.05, 0.5][i % 3], rng.integers(-127, 128, n), 0)
        scans.append(d.astype(np.int16))
    pays = RC.encode_scans(scans)
    assert pays == [R.encode_scan(s) for s in scans]
    back = RC.decode_scans(pays, 5000)
    for a, b in zip(back, scans):
        assert np.array_equal(a, b)


def test_dense_noisy_scan_matches_oracle(rng):
    # a dense residual (noisy content): >50k symbols, model halving many times
    n = 120_000
    d = np.where(rng.random(n) < 0.6, rng.integers(-40, 41, n), 0).astype(np.int16)
    pay = RC.encode_scan(d)
    assert pay == R.encode_scan(d)
    assert np.array_equal(RC.decode_scan(pay, n), d)


def test_parallel_encoder_chunk_edges(rng):
    """The parallel-model encoder (4096-entry scan chunks, <= 1024-symbol model
    steps, halving events between steps) on scans built to hit its seams:
    non-zeros on and either side of chunk boundaries, zero runs spanning whole
    chunks (runs of 255-symbols), an all-zero scan (EOS only), one non-zero
    at the very end, and a dense scan long enough to halve the model."""
    n = 3 * 4096 + 777
    scans = [np.zeros(n, np.int16) for _ in range(6)]
    for j in (0, 4095, 4096, 4097, 8191, 8192, n - 1):
        scans[0][j] = (-1) ** j * (1 + j % 127)
    scans[1][[5, 9000, n - 2]] = [7, -3, 127]            # runs across chunks
    scans[3][n - 1] = -127
    scans[4][:] = np.where(rng.random(n) < 0.9, rng.integers(-127, 128, n), 0)
    scans[5][::256] = 1                                 # gaps of exactly 255
    pays = RC.encode_scans(scans)
    assert pays == [R.encode_scan(s) for s in scans]
    for a, b in zip(RC.decode_scans(pays, n), scans):
        assert np.array_equal(a, b)
    big = np.where(rng.random(300_000) < 0.45, rng.integers(-127, 128, 300_000), 0)
    big = big.astype(np.int16)                          # ~270k symbols: 7+ halvings
    assert RC.encode_scan(big) == R.encode_scan(big)


# ---------------------------------------------------------------------------
# pkg/tests/test_rangecoder.py

def test_symbol_mapping_bijection_and_validation():
    seen = set()
    for k in range(1, 256):
        assert RC.symbol_kind(RC.zero_run_symbol(k)) == ("run", k)
        seen.add(k)
    for v in list(range(-127, 0)) + list(range(1, 128)):
        sym = RC.value_symbol(v)
        assert RC.symbol_kind(sym) == ("value", v)
        seen.add(sym)
    seen.add(RC.EOS)
    assert seen == set(range(RC.ALPHABET_SIZE))
    for bad in (lambda: RC.zero_run_symbol(0), lambda: RC.zero_run_symbol(256),
                lambda: RC.value_symbol(0), lambda: RC.value_symbol(128),
                lambda: RC.validate_stream([RC.EOS, RC.value_symbol(3)]),
                lambda: RC.validate_stream([RC.value_symbol(3)])):
        with pytest.raises(ValueError):
            bad()


def test_scan_symbol_roundtrip_and_long_runs(rng):
    for _ in range(20):
        n = int(rng.integers(0, 2000))
        dense = rng.integers(-127, 128, size=n).astype(np.int16)
        dense[rng.random(n) < 0.8] = 0
        syms = RC.scan_to_symbols(dense)
        RC.validate_stream(syms)
        assert syms == R.scan_to_symbols(dense)
        assert np.array_equal(RC.symbols_to_scan(syms, n), dense)
    dense = np.zeros(1000, np.int16)
    dense[999] = 5
    syms = RC.scan_to_symbols(dense)
    assert syms[:3] == [255, 255, 255] and RC.symbol_kind(syms[3]) == ("run", 234)


def test_roundtrips():
    assert len(RC.encode_stream([RC.EOS])) <= 8
    assert RC.decode_stream(RC.encode_stream([RC.EOS])) == [RC.EOS]
    dense = np.zeros(10_000, np.int16)
    data = RC.encode_scan(dense)
    assert len(data) <= 200 and np.array_equal(RC.decode_scan(data, 10_000), dense)
    syms = [RC.value_symbol(127), RC.value_symbol(-127)] * 500 + [RC.EOS]
    assert RC.decode_stream(RC.encode_stream(syms)) == syms


def test_random_streams_batch(rng):
    streams = [[int(rng.integers(1, RC.ALPHABET_SIZE)) for _ in range(int(rng.integers(0, 120)))]
               + [RC.EOS] for _ in range(200)]
    datas = RC.encode_symbol_streams(streams)
    for s, d in zip(streams, datas):
        assert d == R.encode_stream(s)
    for s, d in zip(streams[:20], datas[:20]):
        assert RC.decode_stream(d) == s


def test_truncated_input_raises(rng):
    syms = [RC.value_symbol(int(v)) for v in rng.integers(1, 100, size=200)] + [RC.EOS]
    data = RC.encode_stream(syms)
    with pytest.raises(RC.CorruptStreamError):
        RC.decode_stream(data[:len(data) // 2])
    with pytest.raises(RC.CorruptStreamError):
        RC.decode_stream(b"")
    with pytest.raises(RC.CorruptStreamError):
        RC.symbols_to_scan([RC.zero_run_symbol(100), RC.EOS], 50)


def test_compression_tracks_entropy(rng):
    probs = {1: 0.5, -1: 0.25, 2: 0.125, -2: 0.125}
    h = -sum(p * math.log2(p) for p in probs.values())
    n = 100_000
    vals = rng.choice(list(probs), size=n, p=list(probs.values()))
    syms = [RC.value_symbol(int(v)) for v in vals] + [RC.EOS]
    data = RC.encode_stream(syms)
    assert len(data) * 8 / (h * n) == pytest.approx(1.0, abs=0.05)
    assert RC.decode_stream(data) == syms


def test_sub_bit_symbols_decode():
    # the adaptive model codes a long constant run in far under one bit per
    # symbol (20001 symbols in ~436 bytes): the decoder's output buffer must
    # not be sized from the byte count
    syms = [255] * 20000 + [RC.EOS]
    data = RC.encode_stream(syms)
    assert data == R.encode_stream(syms)
    assert len(data) * 8 < len(syms)
    assert RC.decode_stream(data) == syms
    with pytest.raises(RC.CorruptStreamError):
        RC.decode_stream(data, max_symbols=1000)


# ---------------------------------------------------------------------------
# pkg/tests/test_residual.py (core properties)

def test_residual_properties(rng):
    avg = rng.standard_normal((16, 16, 3)) * 0.05
    sr = RS.sparsify_quantize(avg, theta=0.02)
    deq = sr.qvalues.astype(np.float64) * sr.quant_step
    assert (np.abs(deq) >= 0.02).all()
    assert np.all(np.abs(avg.ravel()[sr.indices] - deq) <= sr.quant_step / 2 + 1e-12)
    with pytest.raises(ValueError):
        RS.sparsify_quantize(avg, theta=-1.0)
    with pytest.raises(ValueError):
        RS.sparsify_quantize(avg, quant_step=0.0)
    # a missing residual leaves the reconstruction untouched
    g = V.GoP(0, tuple(V.Frame(np.full((16, 16, 3), 0.5, np.float32)) for _ in range(9)))
    assert RS.apply_residual(g, None) is g
    ap = RS.apply_residual(g, sr)
    assert np.array_equal(ap.frames[0].samples,
                          R.apply(np.full((16, 16, 3), 0.5, np.float32),
                                  R.dense_delta(sr.indices, sr.qvalues, sr.quant_step, (16, 16, 3))))
    assert RS.raw_residual_rate(1920, 1080, 30) == 1920 * 1080 * 3 * 8 * 30


@pytest.mark.parametrize("H,W,s", [(270, 480, 3), (73, 101, 2), (61, 97, 3), (120, 200, 2)])
def test_encode_work_output_equals_downscale(H, W, s):
    """K1's optional working-frame output (sst_encode_work) is scale_gop(down)
    bit for bit (the standalone sst_downscale kernel, itself golden-checked),
    tokens are unchanged by asking for it; odd sizes exercise the edge
    replication and the block padding that must not be written."""
    import torch
    from paper_2602_03529_b200 import _dev, _lib
    from paper_2602_03529_b200.pipeline import GopCodec
    G = 2
    gen = torch.Generator(device="cuda").manual_seed(3)
    frames = torch.rand((G, 9, H, W, 3), generator=gen, device="cuda")
    c = GopCodec(G, H, W, s)
    c.encode(frames, G, 0)
    tok0 = c.tok.clone()
    h, w = -(-H // s), -(-W // s)
    work = torch.full((G, 9, h, w, 3), -7.0, device="cuda")
    c.encode(frames, G, 0, work=work)
    ref = torch.empty_like(work)
    _lib.call("sst_downscale", frames.data_ptr(), G * 9, H, W, s, ref.data_ptr(), _dev.stream())
    torch.cuda.synchronize()
    assert torch.equal(c.tok, tok0)
    assert torch.equal(work, ref)
