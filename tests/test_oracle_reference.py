"""CPU: differential test of the oracle against the LIVE reference package on
many seeded, adversarial inputs.  Runs only where /root/reference exists (the
build container); the golden fixtures carry the same evidence elsewhere."""

import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import semstream_oracle as O

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="live reference not mounted")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, str(REF))
    import semstream.codec as C
    import semstream.selection as S
    import semstream.transport as T
    import semstream.video as V
    return C, S, T, V


def _bits(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a, b) and \
        np.array_equal(np.signbit(a), np.signbit(b))


def _adversarial_frames(rng, n, h, w):
    """float32 samples in [0, 1] with a wide exponent spread, exact zeros,
    exact ones and dyadic values."""
    e = rng.integers(-40, 1, (n, h, w, 3)).astype(np.float64)
    a = rng.random((n, h, w, 3)) * 2.0 ** e
    pick = rng.random((n, h, w, 3))
    a = np.where(pick < 0.05, 0.0, a)
    a = np.where((pick >= 0.05) & (pick < 0.08), 1.0, a)
    a = np.where((pick >= 0.08) & (pick < 0.2), np.floor(rng.random((n, h, w, 3)) * 256) / 256, a)
    return np.clip(a, 0, 1).astype(np.float32)


def test_downscale_and_encode_adversarial(ref):
    C, S, T, V = ref
    rng = np.random.default_rng(11)
    for trial in range(12):
        h, w = (int(x) for x in rng.integers(3, 70, 2))
        frames = _adversarial_frames(rng, 9, h, w)
        gop = V.GoP(0, tuple(V.Frame(f) for f in frames))
        for s in (2, 3):
            work = C.scale_gop(gop, s, "down")
            ours = O.downscale(frames, s)
            assert _bits(ours, np.stack([f.samples for f in work.frames]))
            I, P = C.encode_gop(work, C.CodecConfig())
            oi, op = O.encode(ours)
            assert _bits(oi, I.values) and _bits(op, P.values)
            assert _bits(O.similarity(op, oi), S.token_similarity(P, I).values)


def test_similarity_and_topk_with_ties(ref):
    C, S, T, V = ref
    rng = np.random.default_rng(12)
    for trial in range(20):
        h, w = (int(x) for x in rng.integers(1, 20, 2))
        i = rng.standard_normal((h, w, 12))
        p = rng.standard_normal((h, w, 12))
        sel = rng.random((h, w)) < 0.4
        p[sel] = i[sel] * rng.choice([1.0, 2.5, -1.0])       # exact +-1 ties
        p[rng.random((h, w)) < 0.1] = 0.0                   # zero-norm rules
        i[rng.random((h, w)) < 0.05] = 0.0
        tp = C.TokenMatrix("P", p, np.ones((h, w), bool))
        ti = C.TokenMatrix("I", i, np.ones((h, w), bool))
        sim = S.token_similarity(tp, ti)
        ours = O.similarity(p, i)
        assert _bits(ours, sim.values)
        for rate in (0.0, 0.05, 0.1, 0.25, 0.3):
            assert np.array_equal(O.top_k_mask(ours, O.drop_count(rate, ours.size)),
                                  S.build_drop_mask(sim, rate))


def test_packetize_parse_reassemble(ref):
    C, S, T, V = ref
    rng = np.random.default_rng(13)
    for trial in range(25):
        h, w = (int(x) for x in rng.integers(1, 12, 2))
        c = int(rng.choice([1, 2, 3, 12]))
        vals = rng.uniform(-4, 4, (h, w, c)) * rng.choice([1.0, 1e-6, 1e3])
        mask = rng.random((h, w)) > rng.choice([0.0, 0.3, 1.0])
        vals[rng.random((h, w)) < 0.2] = 1.234               # constant-ish rows
        vals = np.where(mask[..., None], vals, 0.0)
        kind = "I" if trial % 2 else "P"
        m = C.TokenMatrix(kind, vals, mask, gop_id=trial)
        scale = int(rng.choice([1, 2, 3]))
        ref_wire = [p.to_bytes() for p in T.packetize_tokens(m, scale=scale)]
        ours = O.packetize(O.KIND_I if kind == "I" else O.KIND_P, trial, vals, mask, scale)
        assert ours == ref_wire
        keep = [d for d in ref_wire if rng.random() > 0.3]
        keep = keep + keep[:2]                                # duplicates
        st_ref, st_or = {}, {}
        back = T.reassemble([T.parse_packet(d) for d in keep], (h, w, c), kind, trial,
                            stats=st_ref)
        ov, om = O.reassemble([O.parse(d) for d in keep], (h, w, c), stats=st_or)
        assert _bits(ov, back.values) and np.array_equal(om, back.mask)
        assert st_or == st_ref


def test_decode_upscale_blend(ref):
    C, S, T, V = ref
    rng = np.random.default_rng(14)
    cfg = C.CodecConfig()
    for trial in range(10):
        h, w = (int(x) for x in rng.integers(5, 40, 2))
        ht, wt = -(-h // 8), -(-w // 8)
        iv = rng.standard_normal((ht, wt, 12)) * 2 + np.tile([4, 0, 0, 0], 3)
        pv = rng.standard_normal((ht, wt, 12)) * 2 + np.tile([4, 0, 0, 0], 3)
        pm = rng.random((ht, wt)) > 0.3
        pv = np.where(pm[..., None], pv, 0.0)
        I = C.TokenMatrix("I", iv, np.ones((ht, wt), bool), frame_shape=(h, w))
        P = C.TokenMatrix("P", pv, pm, frame_shape=(h, w))
        rec = C.decode_gop(I, P, cfg)
        oi, op = O.decode(iv, pv, pm, (h, w))
        assert _bits(oi, rec.frames[0].samples) and _bits(op, rec.frames[1].samples)
        for s in (2, 3):
            crop = (h * s - int(rng.integers(0, s)), w * s - int(rng.integers(0, s)))
            up = C.scale_gop(rec, s, "up", crop=crop)
            assert _bits(O.upscale(oi, s, crop), up.frames[0].samples)
            assert _bits(O.upscale(op, s, crop), up.frames[1].samples)
            prev = V.GoP(0, tuple(V.Frame(x) for x in np.clip(
                rng.random((9,) + up.frames[0].samples.shape), 0, 1).astype(np.float32)))
            for n in (1, 2, 4, 8):
                bl = C.blend_boundary(prev, up, n)
                ours = O.blend([f.samples for f in prev.frames], [f.samples for f in up.frames], n)
                for a, b in zip(ours, bl.frames):
                    assert _bits(a, b.samples)


def test_metrics(ref):
    C, S, T, V = ref
    rng = np.random.default_rng(15)
    for shape in ((16, 24, 3), (45, 80, 3), (1080, 1920, 3)):
        a = _adversarial_frames(rng, 9, *shape[:2])
        b = _adversarial_frames(rng, 9, *shape[:2])
        ga = V.GoP(0, tuple(V.Frame(x, timestamp_index=t) for t, x in enumerate(a)))
        gb = V.GoP(1, tuple(V.Frame(x, timestamp_index=t) for t, x in enumerate(b)))
        assert O.gop_psnr(list(a), list(b)) == V.gop_psnr(ga, gb)
        for n in (1, 2, 5, 9):
            for norm in ("l1", "l2"):
                assert O.boundary_flicker(a, b, n, norm) == V.boundary_flicker(ga, gb, n, norm)
        assert O.inter_frame_consistency(b) == V.inter_frame_consistency(gb.frames)


# ---------------------------------------------------------------------------
# raw-rgb24 file formats (video.py:103-143): the CLI's ingest and egress

def test_rgb24_conversions_match_reference_io(ref, tmp_path):
    """frames_from_rgb24 == load_raw_video's frames and rgb24_from_frames ==
    write_raw_video's bytes on every byte value and on float samples at and
    around the rint ties (v * 255 = k + 1/2)."""
    C, S, T, V = ref
    rng = np.random.default_rng(24)
    H, W = 6, 10
    raw = np.concatenate([np.arange(256, dtype=np.uint8),
                          rng.integers(0, 256, 2 * H * W * 3 - 256, dtype=np.uint8)])
    path = tmp_path / "clip.rgb"
    path.write_bytes(raw.tobytes())
    frames = V.load_raw_video(str(path), W, H)
    got = O.frames_from_rgb24(raw.reshape(2, H, W, 3))
    for t in range(2):
        assert _bits(frames[t].samples, got[t])
    k = rng.integers(0, 255, H * W * 3)
    ties = ((2 * k + 1) / 510.0).astype(np.float32)            # float32 near the k + 1/2 boundary
    vals = np.concatenate([ties, np.nextafter(ties, np.float32(0)), np.nextafter(ties, np.float32(1)),
                           rng.random(H * W * 3, dtype=np.float32)])
    vals = np.clip(vals, 0, 1).astype(np.float32)[: 2 * H * W * 3].reshape(2, H, W, 3)
    out = tmp_path / "out.rgb"
    V.write_raw_video(str(out), [V.Frame(vals[t], timestamp_index=t) for t in range(2)])
    assert out.read_bytes() == O.rgb24_from_frames(vals).tobytes()
