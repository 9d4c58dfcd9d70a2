"""GPU parity against the golden fixtures generated from the live reference
(tests/golden/make_golden.py): every intermediate must be bit-identical."""

import numpy as np
import pytest
import torch

from helpers import digest, golden_cases, case_clip, wire_digest

pytestmark = pytest.mark.gpu

CASES = golden_cases()


def _api_gops(c):
    """The reference composition, through this package's drop-in API."""
    from paper_2602_03529_b200 import codec as C, selection as S, transport as T, video as V
    cc = c["case"]
    clip = case_clip(cc)
    cfg = C.CodecConfig()
    prev = None
    for k, rec in enumerate(c["gops"]):
        s = rec["scale"]
        src = clip.gop(k)
        g = V.GoP(k, tuple(V.Frame(f, timestamp_index=t) for t, f in enumerate(src)))
        work = g if s == 1 else C.scale_gop(g, s, "down")
        I, P = C.encode_gop(work, cfg)
        sim = S.token_similarity(P, I)
        drop = np.zeros(I.mask.shape, dtype=bool)
        if cc["drop"] > 0.0:
            drop = S.build_drop_mask(sim, cc["drop"])
            P = C.apply_token_mask(P, drop)
        wire = [p.to_bytes() for p in T.packetize_tokens(I, scale=s) + T.packetize_tokens(P, scale=s)]
        lost = set(rec["lost"])
        recv = T.parse_packets([d for j, d in enumerate(wire) if j not in lost])
        shape = I.values.shape
        st_i, st_p = {}, {}
        ri = T.reassemble([p for p in recv if p.kind == "I"], shape, "I", gop_id=k,
                          frame_shape=I.frame_shape, stats=st_i)
        rp = T.reassemble([p for p in recv if p.kind == "P"], shape, "P", gop_id=k,
                          frame_shape=I.frame_shape, stats=st_p)
        dec = C.decode_gop(ri, rp, cfg)
        up = dec if s == 1 else C.scale_gop(dec, s, "up", crop=(cc["H"], cc["W"]))
        if prev is not None:
            up = C.blend_boundary(prev, up, 2)
        prev = up
        yield rec, dict(src=src, work=work.stacked(), I=I, P=P, sim=sim.values, drop=drop,
                        wire=wire, dec=dec, out=up.stacked(),
                        rows=[st_i["rows_received"], st_p["rows_received"]])


@pytest.mark.parametrize("c", CASES, ids=[c["case"]["name"] for c in CASES])
def test_api_pipeline_matches_reference(c):
    for rec, r in _api_gops(c):
        assert digest(r["src"]) == rec["src"]
        assert digest(r["work"]) == rec["work"]
        assert digest(r["I"].values) == rec["tok_i"]
        assert digest(r["sim"]) == rec["sim"]
        assert digest(r["drop"].astype(np.uint8)) == rec["drop"]
        assert digest(r["P"].values) == rec["tok_p"]
        assert digest(r["P"].mask.astype(np.uint8)) == rec["p_mask"]
        assert wire_digest(r["wire"]) == rec["wire"]
        assert r["rows"] == rec["rows_received"]
        assert digest(r["dec"].frames[0].samples) == rec["i_img"]
        assert digest(r["dec"].frames[1].samples) == rec["p_img"]
        assert digest(r["out"]) == rec["out"]
        # a19: the GPU metric path reproduces the reference's gop_psnr exactly
        # (numpy pairwise summation order, csrc/metrics.cu)
        from paper_2602_03529_b200 import video as V
        src = V.GoP(0, tuple(V.Frame(f, timestamp_index=t) for t, f in enumerate(r["src"])))
        out = V.GoP(0, tuple(V.Frame(f, timestamp_index=t) for t, f in enumerate(r["out"])))
        assert V.gop_psnr(src, out) == (rec["psnr_db"], rec["mse"])


BATCH_CASES = [c for c in CASES if all(g["scale"] in (2, 3) for g in c["gops"])]


@pytest.mark.parametrize("c", BATCH_CASES, ids=[c["case"]["name"] for c in BATCH_CASES])
def test_batched_pipeline_matches_reference(c):
    """The fused device path (StreamBank / GopCodec: K1..K5) on one stream."""
    from paper_2602_03529_b200.pipeline import StreamBank
    cc = c["case"]
    clip = case_clip(cc)
    bank = StreamBank(1, cc["H"], cc["W"])
    for k, rec in enumerate(c["gops"]):
        s = rec["scale"]
        frames = torch.from_numpy(clip.gop(k)[None].copy()).cuda()
        out = torch.empty_like(frames)
        codec = bank.codecs[s]
        present = torch.ones(codec.n_pkt_per_gop, dtype=torch.uint8, device="cuda")
        if rec["lost"]:
            present[torch.tensor(rec["lost"], device="cuda")] = 0
        bank.step({s: frames}, {s: out}, {s: [0]}, {s: [k]}, drop_rate=cc["drop"],
                  present_by_scale={s: present})
        torch.cuda.synchronize()
        arena = codec.arena.cpu().numpy()
        lengths = codec.lengths.cpu().numpy()
        wire = [arena[j, :lengths[j]].tobytes() for j in range(codec.n_pkt_per_gop)]
        assert wire_digest(wire) == rec["wire"]
        assert digest(codec.tok[0, 0].cpu().numpy()) == rec["tok_i"]
        assert digest(codec.tok[0, 1].cpu().numpy()) == rec["tok_p"]
        assert digest(codec.sim[0].cpu().numpy()) == rec["sim"]
        img = codec.img[(bank.step_idx - 1) & 1][0].cpu().numpy()
        assert digest(img[0]) == rec["i_img"]
        assert digest(img[1]) == rec["p_img"]
        assert digest(out[0].cpu().numpy()) == rec["out"]
        from paper_2602_03529_b200.video import gop_psnr_device
        assert gop_psnr_device(frames[0], out[0]) == (rec["psnr_db"], rec["mse"])
        st = codec.stats[:4].cpu().numpy()
        assert [int(st[1]), int(st[3])] == rec["rows_received"]
