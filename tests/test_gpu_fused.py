"""GPU: the decoder-fused reconstruction (SURVEY §8 a15-a18 in one kernel):
``sst_unpack_tokens`` stops the receiver at the dequantised token matrices
and ``sst_upscale_blend_tok`` runs decode_gop's IDCT, clip and I-concealment
(codec.py:131-140,160-186) for exactly the working-image windows it upscales
and blends (codec.py:217-296), including the previous GoP's P window from its
own tokens.  Checked bit for bit against the oracle pipeline and against the
unfused kernels (sst_unpack_decode + sst_upscale_blend) -- many streams,
variable scale per GoP (the previous window at another scale), every blend
width, intelligent drop, network loss (concealment of lost P rows, zeroed
lost I rows), corrupted packets and 1080p."""

import numpy as np
import pytest
import torch

from oracle import semstream_oracle as O
from oracle.synth import make_clip
from paper_2602_03529_b200 import _dev, _lib
from paper_2602_03529_b200.pipeline import GopCodec, StreamBank

pytestmark = pytest.mark.gpu


def _wire(codec, g):
    arena = codec.arena.cpu().numpy()
    lengths = codec.lengths.cpu().numpy()
    n = codec.n_pkt_per_gop
    return [[arena[i * n + j, :lengths[i * n + j]].tobytes() for j in range(n)] for i in range(g)]


@pytest.mark.parametrize("blend_n", [1, 2, 3, 4, 6])
@pytest.mark.parametrize("HW", [(72, 96), (60, 70), (47, 58)])
def test_fused_multistream_variable_scale_matches_oracle(blend_n, HW):
    H, W = HW
    n_streams, n_gops = 4, 3
    clips = [make_clip("noisy-motion" if i % 2 else "moving-square", W, H, 9 * n_gops, seed=10 + i)
             for i in range(n_streams)]
    sched = [[(3, 2, 3), (2, 2, 3), (3, 3, 2), (2, 3, 2)][i] for i in range(n_streams)]
    fused = StreamBank(n_streams, H, W, blend_n=blend_n, fused=True)
    plain = StreamBank(n_streams, H, W, blend_n=blend_n)
    assert fused.fused
    prev = [None] * n_streams
    for k in range(n_gops):
        by_s = {}
        for i in range(n_streams):
            by_s.setdefault(sched[i][k], []).append(i)
        frames = {s: torch.from_numpy(np.stack([clips[i].gop(k) for i in ids])).cuda()
                  for s, ids in by_s.items()}
        outs_f = {s: torch.full_like(f, -3.0) for s, f in frames.items()}
        outs_p = {s: torch.empty_like(f) for s, f in frames.items()}
        gids = {s: [k] * len(ids) for s, ids in by_s.items()}
        fused.step(frames, outs_f, by_s, gids, drop_rate=0.2)
        plain.step(frames, outs_p, by_s, gids, drop_rate=0.2)
        torch.cuda.synchronize()
        for s, ids in by_s.items():
            got = outs_f[s].cpu().numpy()
            assert np.array_equal(got.view(np.uint32), outs_p[s].cpu().numpy().view(np.uint32)), (k, s)
            wire = _wire(fused.codecs[s], len(ids))
            for j, i in enumerate(ids):
                ref = O.pipeline_gop(clips[i].gop(k), s, gop_id=k, drop_rate=0.2,
                                     prev_out=prev[i], blend_width=blend_n)
                prev[i] = ref["frames"]
                assert wire[j] == ref["wire"], (k, i)
                assert np.array_equal(got[j], np.stack(ref["frames"])), (k, i, s)


@pytest.mark.parametrize("s", [2, 3])
def test_fused_under_packet_loss_and_corruption(s):
    """Lost I rows decode to zero, lost / dropped P rows are concealed by the
    I blocks, a CRC-corrupted packet is rejected -- in the current GoP and in
    the previous one the blend reads."""
    H, W = 64, 96
    n_streams = 3
    clips = [make_clip("moving-square" if i else "noisy-motion", W, H, 18, seed=20 + i)
             for i in range(n_streams)]
    banks = {True: StreamBank(n_streams, H, W, fused=True), False: StreamBank(n_streams, H, W)}
    rng = np.random.default_rng(5 + s)
    prev = [None] * n_streams
    for k in range(2):
        frames = torch.from_numpy(np.stack([c.gop(k) for c in clips])).cuda()
        npk = banks[True].codecs[s].n_pkt_per_gop
        lost_sets = [set(int(j) for j in np.flatnonzero(rng.random(npk) < 0.3)) for _ in range(n_streams)]
        present = torch.tensor([0 if j in lost_sets[i] else 1 for i in range(n_streams) for j in range(npk)],
                               dtype=torch.uint8, device="cuda")
        outs = {}
        for fz, bank in banks.items():
            out = torch.empty_like(frames)
            bank.step({s: frames}, {s: out}, {s: list(range(n_streams))}, {s: [k] * n_streams},
                      drop_rate=0.1, present_by_scale={s: present})
            outs[fz] = out
        torch.cuda.synchronize()
        got = outs[True].cpu().numpy()
        assert np.array_equal(got.view(np.uint32), outs[False].cpu().numpy().view(np.uint32)), k
        for i in range(n_streams):
            ref = O.pipeline_gop(clips[i].gop(k), s, gop_id=k, drop_rate=0.1, lost=lost_sets[i],
                                 prev_out=prev[i], blend_width=2)
            prev[i] = ref["frames"]
            assert np.array_equal(got[i], np.stack(ref["frames"])), (k, i)


def test_fused_entry_points_direct():
    """sst_unpack_tokens' matrices are TokenPacket.dequantized scattered by
    reassemble (zeros where missing), and sst_upscale_blend_tok equals
    sst_unpack_decode + sst_upscale_blend on the same packets, with a
    corrupted P packet."""
    H, W, s = 48, 64, 2
    src = make_clip("moving-square", W, H, 9, seed=31).gop(0)
    c = GopCodec(1, H, W, s)
    c.set_gop_ids([0])
    c.encode(torch.from_numpy(src[None].copy()).cuda(), 1, c.drop_k(0.2))
    torch.cuda.synchronize()
    victim = c.Ht + 2
    c.arena[victim, 40] ^= 0x5A
    img = c.decode(1, 0).clone()
    c.decode(1, 1, fused=True)
    torch.cuda.synchronize()
    ref = O.pipeline_gop(src, s, gop_id=0, drop_rate=0.2, lost={victim})
    tok = c.tokq[1][0].cpu().numpy()
    pv = c.pvalid[1][0].cpu().numpy()
    assert np.array_equal(img.cpu().numpy()[0, 0], ref["i_img"])
    assert pv[victim - c.Ht].sum() == 0                    # the corrupted P row is all invalid
    out_a = torch.empty((1, 9, H, W, 3), device="cuda")
    out_b = torch.full((1, 9, H, W, 3), -1.0, device="cuda")
    c.reconstruct(1, 0, out_a)
    c.reconstruct(1, 1, out_b, fused=True)
    torch.cuda.synchronize()
    assert np.array_equal(out_a.cpu().numpy().view(np.uint32), out_b.cpu().numpy().view(np.uint32))
    assert np.array_equal(out_b.cpu().numpy()[0], np.stack(ref["frames"]))
    assert np.isfinite(tok).all()


def test_fused_1080p_equals_unfused():
    H, W = 1080, 1920
    clip = make_clip("moving-square", W, H, 18, seed=2)
    banks = {fz: StreamBank(2, H, W, fused=fz) for fz in (True, False)}
    for k, s in enumerate((3, 2)):
        frames = torch.from_numpy(np.stack([clip.gop(k), clip.gop(1 - k)])).cuda()
        outs = {}
        for fz, bank in banks.items():
            outs[fz] = torch.empty_like(frames)
            bank.step({s: frames}, {s: outs[fz]}, {s: [0, 1]}, {s: [k, k]}, drop_rate=0.1)
        torch.cuda.synchronize()
        assert torch.equal(outs[True].view(torch.int32), outs[False].view(torch.int32)), k


def test_fused_rejects_uint8_output():
    H, W = 48, 64
    bank = StreamBank(1, H, W, fused=True)
    frames = torch.zeros((1, 9, H, W, 3), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError, match="float32"):
        bank.step({3: frames}, {3: torch.empty_like(frames)}, {3: [0]}, {3: [0]})
