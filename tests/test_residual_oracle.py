"""CPU: the residual / range-coder oracle (oracle/residual_oracle.py) pinned
against fixtures generated from the live reference."""

import numpy as np
import pytest

from helpers import digest
from oracle import residual_oracle as R
from oracle import semstream_oracle as O
from oracle.synth import make_clip
from residual_helpers import avg_input, golden, symbol_stream

G = golden()


@pytest.mark.parametrize("c", G["cases"], ids=[str(c["seed"]) for c in G["cases"]])
def test_sparsify_encode_fit_match_reference(c):
    avg = avg_input(c["seed"], c["shape"], c["scale"])
    idx, qv = R.sparsify(avg)
    assert digest(idx) == c["indices"] and digest(qv) == c["qvalues"]
    dense = np.zeros(avg.size, np.int16)
    dense[idx] = qv
    payload = R.encode_scan(dense)
    assert digest(payload) == c["payload"]
    assert np.array_equal(R.decode_scan(payload, avg.size), dense)
    for f in c["fits"]:
        ind, q, pay, theta = R.fit_to_budget(avg, f["budget"])
        assert (ind is None) == f["none"]
        assert digest(pay) == f["payload"] and theta == f["theta"]
        if ind is not None:
            assert digest(ind) == f["indices"] and digest(q) == f["qvalues"]


@pytest.mark.parametrize("s", G["streams"], ids=[str(s["seed"]) for s in G["streams"]])
def test_range_coder_streams_match_reference(s):
    syms = symbol_stream(s["seed"], s["n"])
    data = R.encode_stream(syms)
    assert digest(data) == s["data"] and len(data) == s["len"]
    assert R.decode_stream(data) == syms


def test_session_residual_matches_reference():
    s = G["session"]
    src = make_clip(s["clip"], s["W"], s["H"], 9, seed=s["seed"]).gop(0)
    work = O.downscale(src, s["scale"])
    i_vals, p_vals = O.encode(work)
    i_img, p_img = O.decode(i_vals, p_vals, np.ones(i_vals.shape[:2], bool), work.shape[1:3])
    recon = np.stack([i_img] + [p_img] * 8)
    res = R.compute_residual(work, recon)
    assert digest(res) == s["residual"]
    avg = R.aggregate(res)
    assert digest(avg) == s["avg"]
    ind, q, pay, theta = R.fit_to_budget(avg, s["budget"])
    assert digest(ind) == s["indices"] and digest(pay) == s["payload"] and theta == s["theta"]
    delta = R.dense_delta(ind, q, R.DEFAULT_QUANT_STEP, avg.shape)
    applied = np.stack([R.apply(i_img, delta)] + [R.apply(p_img, delta)] * 8)
    assert digest(applied) == s["applied"]


def test_truncation_and_overrun_errors():
    data = R.encode_stream([383 + 5] * 200 + [0])
    with pytest.raises(R.OracleStreamError):
        R.decode_stream(data[:len(data) // 2])
    with pytest.raises(R.OracleStreamError):
        R.decode_stream(b"")
    with pytest.raises(R.OracleStreamError):
        R.symbols_to_scan([100, 0], 50)
