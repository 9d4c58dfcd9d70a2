"""GPU: this package as a drop-in INSIDE the unmodified reference session
(SURVEY §8 rows b and f3).

The reference package is installed, unmodified, in the git-ignored
``baseline/_ref`` (``pip install --no-deps --target baseline/_ref`` of a copy
of /root/reference/pkg; it travels to the GPU box with the snapshot).  Two
ways in:

* the plug-in point -- ``SessionConfig.tokenizer_encode / tokenizer_decode``
  (session.py:57-61, consumed at session.py:117-118,140,186,227,336; contract
  pinned by pkg/tests/test_session.py:151-182);
* the module-level hot path -- scale_gop, encode/decode, similarity, drop
  mask, apply mask, packetise, reassemble, blend and the residual layer
  swapped for this package's functions in the reference session's (and
  GopAssembly's) namespaces.

Either way the virtual-clock session must be byte-for-byte the stock one:
identical event-log rows and identical GopRecords (PSNR floats included).
Acceptance gates #4, #5 and #9 (pkg/tests/test_acceptance.py) then run with
the GPU codec in place.
"""

import os
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
if not (REF / "semstream" / "__init__.py").is_file():
    pytest.skip("baseline/_ref (the reference install) is absent", allow_module_level=True)
if str(REF) not in sys.path:
    sys.path.insert(0, str(REF))

import semstream.session as RS                     # noqa: E402  (the reference)
import semstream.transport as RT                   # noqa: E402
from semstream.netem import constant_trace, save_trace, square_wave_trace  # noqa: E402
from semstream.ratecontrol import Mode               # noqa: E402
from semstream.report import tracking_stats        # noqa: E402
from semstream.session import SessionConfig, run_streaming_session  # noqa: E402
from semstream.synth import MovingSquareClip, NoisyMotionClip  # noqa: E402

import paper_2602_03529_b200 as B                  # noqa: E402
from paper_2602_03529_b200 import codec as BC, rangecoder as BRC, residual as BR  # noqa: E402
from paper_2602_03529_b200 import selection as BS, transport as BT  # noqa: E402


def _session(loss=0.0, seed=1, frames=54, rate=2_000_000, clip=None, **kw):
    clip = clip or MovingSquareClip(160, 128, frames, seed=2)
    cfg = SessionConfig(clip=clip, trace=constant_trace(rate), loss_rate=loss, seed=seed, **kw)
    return run_streaming_session(cfg)


def _plugged(**kw):
    return _session(tokenizer_encode=B.tokenizer_encode, tokenizer_decode=B.tokenizer_decode, **kw)


def _same(a, b):
    assert a.log.rows == b.log.rows
    assert a.records == b.records                  # GopRecord dataclass equality (floats exact)
    assert a.rendered_frames == b.rendered_frames


def _swap_hot_path(monkeypatch, residual=True):
    """Swap the reference session's (and GopAssembly's) hot-path functions
    for this package's."""
    swaps = [("scale_gop", BC.scale_gop), ("encode_gop", BC.encode_gop),
             ("decode_gop", BC.decode_gop), ("apply_token_mask", BC.apply_token_mask),
             ("blend_boundary", BC.blend_boundary), ("token_similarity", BS.token_similarity),
             ("build_drop_mask", BS.build_drop_mask), ("packetize_tokens", BT.packetize_tokens),
             ("reassemble", BT.reassemble)]
    if residual:
        swaps += [("residual_mod", BR), ("CorruptStreamError", BRC.CorruptStreamError)]
    for name, fn in swaps:
        monkeypatch.setattr(RS, name, fn)
    monkeypatch.setattr(RT, "reassemble", BT.reassemble)      # GopAssembly.assemble


@pytest.mark.parametrize("loss,seed", [(0.0, 1), (0.25, 33), (0.25, 9)])
def test_plugin_session_byte_identical(loss, seed):
    _same(_session(loss=loss, seed=seed), _plugged(loss=loss, seed=seed))


# two regimes of the reference's rate controller: 600 kb/s on a noisy clip
# (ExtremeLow: s=3 with intelligent P-token drops, 15 % loss) and 3 Mb/s
# starting in Sufficient (s=2 with residual packets: fit_to_budget + range
# coder, and the encoder-side proxy decode of session.py:178-186)
_REGIMES = {
    "drops": dict(loss=0.15, seed=21, rate=600_000, playout_offset_ms=400.0),
    "residuals": dict(loss=0.1, seed=5, rate=3_000_000, playout_offset_ms=400.0,
                      initial_mode=Mode.SUFFICIENT),
}


def _check_regime(name, res):
    if name == "drops":
        assert any(r.drop_rate > 0 for r in res.records)
    else:
        assert any(r[1] == "send" and r[3] == "R" for r in res.log.rows)


@pytest.mark.parametrize("name", sorted(_REGIMES))
def test_plugin_session_rate_regimes(name):
    kw = dict(_REGIMES[name], clip=NoisyMotionClip(160, 128, 81, seed=4))
    stock, gpu = _session(**kw), _plugged(**kw)
    _same(stock, gpu)
    _check_regime(name, gpu)


def test_plugin_contract_custom_tokenizer_shape():
    # pkg/tests/test_session.py:151-182 with this package's pair
    clip = MovingSquareClip(160, 128, 27, seed=2)
    res = run_streaming_session(SessionConfig(
        clip=clip, trace=constant_trace(2_000_000), seed=1,
        tokenizer_encode=B.tokenizer_encode, tokenizer_decode=B.tokenizer_decode))
    assert len(res.records) == clip.gop_count
    assert all(r.rows_lost == 0 for r in res.records)


@pytest.mark.parametrize("name", sorted(_REGIMES))
def test_whole_hot_path_swapped_into_reference_session(name, monkeypatch):
    kw = dict(_REGIMES[name], clip=NoisyMotionClip(160, 128, 81, seed=4))
    stock = _session(**kw)
    _swap_hot_path(monkeypatch)
    gpu = _session(**kw)
    _same(stock, gpu)
    _check_regime(name, gpu)


# ---------------------------------------------------------------------------
# pkg/tests/test_acceptance.py gates with the GPU codec in the session

def test_acceptance_4_loss_resilience_480p_25pct_gpu():
    import time
    t0 = time.time()
    clip = MovingSquareClip(640, 480, 900, seed=6)
    res = _plugged(loss=0.25, seed=17, rate=5_000_000, clip=clip)
    elapsed = time.time() - t0
    assert res.rendered_fps >= 0.95 * 30.0
    assert res.delay_fraction_within(150.0) >= 0.90
    assert elapsed < 300.0


def test_acceptance_5_bitrate_tracking_square_wave_gpu():
    clip = NoisyMotionClip(320, 240, 2700, seed=3)
    trace = square_wave_trace(200_000, 500_000, 30_000)
    cfg = SessionConfig(clip=clip, trace=trace, loss_rate=0.0, seed=11,
                        playout_offset_ms=1300.0, queue_bytes=40_000,
                        tokenizer_encode=B.tokenizer_encode, tokenizer_decode=B.tokenizer_decode)
    stats = tracking_stats(run_streaming_session(cfg), trace)
    assert stats["tracked_fraction"] >= 0.90
    assert stats["worst_overshoot"] <= 1.05


def test_acceptance_9_stream_determinism_gpu(tmp_path, monkeypatch):
    # `semstream stream` (cli.py) with the session's codec path on the GPU:
    # two seeded runs byte-identical to each other AND to the stock CLI run
    from semstream.cli import main
    trace_path = str(tmp_path / "link.trace")
    save_trace(trace_path, constant_trace(1_500_000))

    def run(name):
        out_dir = str(tmp_path / name)
        rc = main(["stream", "synth:moving-square:160x128:54:seed=2", "--trace", trace_path,
                   "--seed", "21", "--loss-rate", "0.15", "--out-dir", out_dir, "--no-figures"])
        assert rc == 0
        return tuple(open(os.path.join(out_dir, f), "rb").read()
                     for f in ("metrics.csv", "events.csv"))

    stock = run("stock")
    _swap_hot_path(monkeypatch)
    a, b = run("gpu1"), run("gpu2")
    assert a == b == stock


# ---------------------------------------------------------------------------
# batched sender / receiver around the reference's netem (netserve.py)

def test_linked_stream_bank_over_reference_netem():
    """Three streams through one batched GPU codec, each over its own
    reference EmulatedLink (loss, queue, trace pacing, propagation delay):
    every reconstruction equals the CPU reference algorithm fed exactly the
    packets the link delivered before the playout deadline."""
    import numpy as np
    import torch
    from semstream.netem import EmulatedLink, constant_trace

    from oracle import semstream_oracle as O
    from oracle.synth import make_clip
    from paper_2602_03529_b200.netserve import LinkedStreamBank

    H, W, n, gops = 72, 96, 3, 4
    links = [EmulatedLink(constant_trace(rate), loss_rate=0.2, seed=10 + i, queue_bytes=q)
             for i, (rate, q) in enumerate(((2_000_000, 60_000), (60_000, 12_000), (25_000, 800)))]
    lb = LinkedStreamBank(n, H, W, links)
    clips = [make_clip("noisy-motion" if i % 2 else "moving-square", W, H, 9 * gops, seed=i)
             for i in range(n)]
    sched = [(3, 2, 2, 3), (2, 2, 3, 3), (3, 3, 3, 2)]
    prev = [None] * n
    saw = {"lost": 0, "queue": 0, "late": 0}
    for k in range(gops):
        by_s = {}
        for i in range(n):
            by_s.setdefault(sched[i][k], []).append(i)
        frames = {s: torch.from_numpy(np.stack([clips[i].gop(k) for i in ids])).cuda()
                  for s, ids in by_s.items()}
        outs = {s: torch.empty_like(f) for s, f in frames.items()}
        delivered = lb.step(frames, outs, by_s, k, drop_rate=0.1)
        torch.cuda.synchronize()
        for s, ids in by_s.items():
            for j, i in enumerate(ids):
                lost = set(int(p) for p in np.flatnonzero(delivered[i] == 0))
                ref = O.pipeline_gop(clips[i].gop(k), s, gop_id=k, drop_rate=0.1, lost=lost,
                                     prev_out=prev[i])
                prev[i] = ref["frames"]
                assert np.array_equal(outs[s][j].cpu().numpy(), np.stack(ref["frames"])), (k, i)
    for st in lb.stats:
        for key in saw:
            saw[key] += st[key]
        assert st["sent"] == st["delivered"] + st["lost"] + st["queue"] + st["late"]
    assert saw["lost"] > 0 and saw["queue"] > 0 and saw["late"] > 0   # the links really interfered
