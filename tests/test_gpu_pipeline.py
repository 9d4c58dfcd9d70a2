"""GPU: the fused batched path (StreamBank / GopCodec, kernels K1-K5) against
the oracle -- many streams at once, variable scale per GoP, every blend width
(1..4 fused into K5, 5..8 blended per stream after it), network loss and duplicates -- plus full-size
(1080p) properties and determinism."""

import numpy as np
import pytest
import torch

from oracle import semstream_oracle as O
from oracle.synth import make_clip
from paper_2602_03529_b200.pipeline import GopCodec, StreamBank

pytestmark = pytest.mark.gpu


def _wire(codec, g):
    arena = codec.arena.cpu().numpy()
    lengths = codec.lengths.cpu().numpy()
    n = codec.n_pkt_per_gop
    return [[arena[i * n + j, :lengths[i * n + j]].tobytes() for j in range(n)] for i in range(g)]


@pytest.mark.parametrize("blend_n", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("HW", [(72, 96), (60, 70)])      # TMA-aligned and not
def test_multistream_variable_scale_matches_oracle(blend_n, HW):
    H, W = HW
    n_streams, n_gops = 4, 3
    clips = [make_clip("noisy-motion" if i % 2 else "moving-square", W, H, 9 * n_gops, seed=i)
             for i in range(n_streams)]
    sched = [[(3, 2, 3), (2, 2, 3), (3, 3, 2), (2, 3, 2)][i] for i in range(n_streams)]
    bank = StreamBank(n_streams, H, W, blend_n=blend_n)
    prev = [None] * n_streams
    for k in range(n_gops):
        by_s = {}
        for i in range(n_streams):
            by_s.setdefault(sched[i][k], []).append(i)
        frames = {s: torch.from_numpy(np.stack([clips[i].gop(k) for i in ids])).cuda()
                  for s, ids in by_s.items()}
        outs = {s: torch.empty_like(f) for s, f in frames.items()}
        bank.step(frames, outs, by_s, {s: [k] * len(ids) for s, ids in by_s.items()},
                  drop_rate=0.2)
        torch.cuda.synchronize()
        for s, ids in by_s.items():
            wire = _wire(bank.codecs[s], len(ids))
            got = outs[s].cpu().numpy()
            for j, i in enumerate(ids):
                ref = O.pipeline_gop(clips[i].gop(k), s, gop_id=k, drop_rate=0.2,
                                     prev_out=prev[i], blend_width=blend_n)
                prev[i] = ref["frames"]
                assert wire[j] == ref["wire"], (k, i)
                assert np.array_equal(got[j], np.stack(ref["frames"])), (k, i, s)


def test_send_receive_split_equals_step():
    """StreamBank.send + receive (the sender and receiver halves, which a
    pipelined caller can interleave: receive GoP k, then send GoP k + 1) give
    the same packets and frames as step(), bit for bit."""
    H, W = 72, 96
    n_streams, n_gops = 3, 3
    clips = [make_clip("noisy-motion" if i % 2 else "moving-square", W, H, 9 * n_gops, seed=i)
             for i in range(n_streams)]
    sched = [(3, 2, 3), (2, 2, 3), (3, 3, 2)]
    a, b = StreamBank(n_streams, H, W), StreamBank(n_streams, H, W)
    pending = None
    outs_b = {}
    for k in range(n_gops + 1):
        if k < n_gops:
            by_s = {}
            for i in range(n_streams):
                by_s.setdefault(sched[i][k], []).append(i)
            frames = {s: torch.from_numpy(np.stack([clips[i].gop(k) for i in ids])).cuda()
                      for s, ids in by_s.items()}
            gids = {s: [k] * len(ids) for s, ids in by_s.items()}
            outs_a = {s: torch.empty_like(f) for s, f in frames.items()}
            a.step(frames, outs_a, by_s, gids, drop_rate=0.2)
        if pending is not None:                      # pipelined: receive k-1 ...
            pk, p_outs_a = pending
            outs_b = {s: torch.empty_like(o) for s, o in p_outs_a.items()}
            b.receive(outs_b)
            torch.cuda.synchronize()
            for s in outs_b:
                assert torch.equal(outs_b[s], p_outs_a[s]), (pk, s)
        if k < n_gops:                               # ... then send k
            b.send(frames, by_s, gids, drop_rate=0.2)
            torch.cuda.synchronize()
            for s, ids in by_s.items():
                assert _wire(a.codecs[s], len(ids)) == _wire(b.codecs[s], len(ids)), (k, s)
            pending = (k, {s: o.clone() for s, o in outs_a.items()})
    with pytest.raises(RuntimeError):
        b.receive(outs_b)                            # nothing pending


def test_loss_and_duplicate_packets_first_wins():
    H, W = 48, 64
    clip = make_clip("moving-square", W, H, 9, seed=3)
    src = clip.gop(0)
    c = GopCodec(1, H, W, 2)
    c.set_gop_ids([0])
    frames = torch.from_numpy(src[None].copy()).cuda()
    c.encode(frames, 1, c.drop_k(0.3))
    torch.cuda.synchronize()
    wire = _wire(c, 1)[0]
    npk = len(wire)
    rng = np.random.default_rng(0)
    lost = set(int(j) for j in np.flatnonzero(rng.random(npk) < 0.3))
    present = torch.tensor([0 if j in lost else 1 for j in range(npk)], dtype=torch.uint8,
                           device="cuda")
    img = c.decode(1, 0, present=present)
    torch.cuda.synchronize()
    ref = O.pipeline_gop(src, 2, gop_id=0, drop_rate=0.3, lost=lost)
    got = img.cpu().numpy()[0]
    assert np.array_equal(got[0], ref["i_img"]) and np.array_equal(got[1], ref["p_img"])
    st = c.stats[:4].cpu().numpy()
    assert [int(st[1]), int(st[3])] == list(ref["rows_received"])
    status = c.packet_status(1)
    assert int((status == 11).sum()) == len(lost)          # SST_PKT_ABSENT


def test_corrupted_packet_is_rejected_and_concealed():
    H, W = 48, 64
    src = make_clip("moving-square", W, H, 9, seed=4).gop(0)
    c = GopCodec(1, H, W, 3)
    c.set_gop_ids([0])
    c.encode(torch.from_numpy(src[None].copy()).cuda(), 1, 0)
    torch.cuda.synchronize()
    victim = c.Ht + 1                                      # a P-row packet
    c.arena[victim, 30] ^= 0xFF                            # payload bit flip -> CRC mismatch
    img = c.decode(1, 0)
    torch.cuda.synchronize()
    status = c.packet_status(1)
    assert status[victim] == 2                             # SST_PKT_CRC
    ref = O.pipeline_gop(src, 3, gop_id=0, lost={victim})
    got = img.cpu().numpy()[0]
    assert np.array_equal(got[1], ref["p_img"])


def test_1080p_properties_and_determinism():
    H, W = 1080, 1920
    clip = make_clip("moving-square", W, H, 9, seed=0)
    src = torch.from_numpy(clip.gop(0)[None].copy()).cuda()
    outs = []
    for _ in range(2):
        bank = StreamBank(1, H, W)
        o = torch.empty_like(src)
        bank.step({2: src}, {2: o}, {2: [0]}, {2: [0]}, drop_rate=0.1)
        torch.cuda.synchronize()
        outs.append(o)
    assert torch.equal(outs[0], outs[1])
    o = outs[0]
    assert float(o.min()) >= 0.0 and float(o.max()) <= 1.0
    for f in range(2, 9):
        assert torch.equal(o[0, f], o[0, 1])               # P reconstruction materialised 8x
    mse = ((o.double() - src.double()) ** 2).mean().item()
    assert 20.0 < 10 * np.log10(1 / mse) < 40.0


@pytest.mark.parametrize("seed", range(12))
def test_random_configuration_sweep(seed):
    """Seeded random geometry / scale / drop / loss / content / GoP batch:
    packet bytes, working images and the 9 reconstructed frames of every GoP
    bit-identical to the oracle (which is pinned to the live reference)."""
    rng = np.random.default_rng(1000 + seed)
    H, W = int(rng.integers(42, 181)), int(rng.integers(42, 261))   # static-detail needs >= 42
    s = int(rng.choice([2, 3]))
    g = int(rng.integers(1, 4))
    drop = float(rng.choice([0.0, 0.05, 0.1, 0.25, 0.3]))
    kinds = ["moving-square", "noisy-motion", "static-detail", "noise-field", "static-gradient"]
    srcs = [make_clip(kinds[int(rng.integers(len(kinds)))], W, H, 9, seed=int(rng.integers(99))).gop(0)
            for _ in range(g)]
    c = GopCodec(g, H, W, s)
    gop_ids = [int(x) for x in rng.integers(0, 2 ** 32 - 1, size=g, dtype=np.uint64)]
    c.set_gop_ids(gop_ids)
    # np.stack keeps the memory order of a transposed clip view: make it C order
    frames = torch.from_numpy(np.ascontiguousarray(np.stack(srcs))).cuda()
    c.encode(frames, g, c.drop_k(drop))
    torch.cuda.synchronize()
    wires = _wire(c, g)
    npk = c.n_pkt_per_gop
    loss = float(rng.choice([0.0, 0.1, 0.3]))
    lost = [set(int(j) for j in np.flatnonzero(rng.random(npk) < loss)) for _ in range(g)]
    present = torch.tensor([0 if j in lost[i] else 1 for i in range(g) for j in range(npk)],
                           dtype=torch.uint8, device="cuda")
    img = c.decode(g, 0, present=present)
    out = torch.empty_like(frames)
    c.reconstruct(g, 0, out)
    torch.cuda.synchronize()
    img, out = img.cpu().numpy(), out.cpu().numpy()
    for i in range(g):
        ref = O.pipeline_gop(srcs[i], s, gop_id=gop_ids[i], drop_rate=drop, lost=lost[i])
        assert wires[i] == ref["wire"], (seed, i)
        assert np.array_equal(img[i, 0], ref["i_img"]) and np.array_equal(img[i, 1], ref["p_img"])
        assert np.array_equal(out[i], np.stack(ref["frames"])), (seed, i, H, W, s)


def test_non_contiguous_frames_are_rejected():
    H, W = 32, 40
    c = GopCodec(1, H, W, 2)
    src = torch.rand((1, 9, W, H, 3), device="cuda").transpose(2, 3)   # [1][9][H][W][3] view
    with pytest.raises(ValueError, match="contiguous"):
        c.encode(src, 1)
    with pytest.raises(ValueError, match="float32"):
        c.encode(src.contiguous().double(), 1)


def test_graphed_codec_matches_eager():
    """CUDA-graph replay of the GoP step == the eager launches (3 GoPs:
    first without blending, then both parities with blending)."""
    from paper_2602_03529_b200.pipeline import GraphedGopCodec
    H, W, s = 72, 96, 3
    clip = make_clip("noisy-motion", W, H, 27, seed=8)
    c = GopCodec(1, H, W, s)
    fr = torch.empty((1, 9, H, W, 3), device="cuda")
    out = torch.empty_like(fr)
    gr = GraphedGopCodec(c, 1, fr, out, drop_k=c.drop_k(0.2))
    prev = None
    for k in range(3):
        fr.copy_(torch.from_numpy(clip.gop(k)[None].copy()))
        gr.step([k])
        torch.cuda.synchronize()
        ref = O.pipeline_gop(clip.gop(k), s, gop_id=k, drop_rate=0.2, prev_out=prev)
        prev = ref["frames"]
        assert np.array_equal(out[0].cpu().numpy(), np.stack(ref["frames"])), k


def test_graphed_stream_bank_matches_eager():
    """GraphedStreamBank (one CUDA-graph replay per GoP, variable scale) is
    bit-identical to the eager StreamBank, blends across scale changes
    included."""
    from paper_2602_03529_b200.pipeline import GraphedStreamBank
    H, W = 72, 96
    clip = make_clip("noisy-motion", W, H, 9 * 7, seed=3)
    sched = (3, 3, 2, 2, 3, 2, 3)
    fr = torch.empty((1, 9, H, W, 3), dtype=torch.float32, device="cuda")
    out_g = torch.empty_like(fr)
    gb = GraphedStreamBank(H, W, fr, out_g, drop_rate=0.2)
    bank = StreamBank(1, H, W)
    out_e = torch.empty_like(fr)
    prev = None
    for k, s in enumerate(sched):
        src = clip.gop(k)
        fr.copy_(torch.from_numpy(src[None].copy()))
        gb.step(s, k)
        bank.step({s: fr}, {s: out_e}, {s: [0]}, {s: [k]}, drop_rate=0.2)
        torch.cuda.synchronize()
        ref = O.pipeline_gop(src, s, gop_id=k, drop_rate=0.2, prev_out=prev)
        prev = ref["frames"]
        assert torch.equal(out_g, out_e), k
        assert np.array_equal(out_g[0].cpu().numpy(), np.stack(ref["frames"])), k
