"""Library baseline for the main path: the proxy codec's per-GoP work written
as plain PyTorch on the GPU (float64 like the reference), at the bench shape
(G x 1080p GoPs per launch, s=3, 10% drop, blend n=2), CUDA-event timed next
to this repository's fused kernels (StreamBank.step) on the same inputs.

The PyTorch version does the same arithmetic classes -- box downscale, the
four-coefficient 8x8 DCT of frame 0 and of the frame 1..8 mean, cosine
similarity, top-k drop, per-row 8-bit quantisation and dequantisation, the
four-coefficient IDCT with concealment, bilinear x s upscale with crop, blend,
clip, float32 -- but no CRC / byte packing, so it does less work than the
fused path.  A comparison, not a parity check.

    python scripts/torch_baseline_proxy.py [G]
"""
import json
import math
import sys

sys.path.insert(0, ".")
import torch
import torch.nn.functional as F

from paper_2602_03529_b200.pipeline import StreamBank

G = int(sys.argv[1]) if len(sys.argv) > 1 else 32
H, W, s, n_blend, drop = 1080, 1920, 3, 2, 0.1
dev = torch.device("cuda")
f64 = torch.float64
h, w = -(-H // s), -(-W // s)
Ht, Wt = -(-h // 8), -(-w // 8)
# orthonormal DCT-II basis rows for the kept zigzag coefficients (0,0),(0,1),(1,0),(2,0)
k = torch.arange(8, dtype=f64, device=dev)
def basis(u):
    c = math.sqrt(1 / 8) if u == 0 else math.sqrt(2 / 8)
    return c * torch.cos((2 * k + 1) * u * math.pi / 16)
B = torch.stack([torch.outer(basis(a), basis(b)) for a, b in ((0, 0), (0, 1), (1, 0), (2, 0))])


def downscale(x):                                   # [N][H][W][3] f32 -> [N][3][h][w] f64
    x = x.permute(0, 3, 1, 2).to(f64)
    x = F.pad(x, (0, w * s - W, 0, h * s - H), mode="replicate")
    return F.avg_pool2d(x, s)


def blocks(img):                                    # [N][3][h][w] -> [N][3][Ht][Wt][8][8]
    img = F.pad(img, (0, Wt * 8 - w, 0, Ht * 8 - h), mode="replicate")
    return img.view(img.shape[0], 3, Ht, 8, Wt, 8).permute(0, 1, 2, 4, 3, 5)


def step(frames, prev_up, out):
    lo = downscale(frames.view(G * 9, H, W, 3)).view(G, 9, 3, h, w)
    imgs = torch.stack([lo[:, 0], lo[:, 1:].mean(1)], 1).view(G * 2, 3, h, w)
    tok = torch.einsum("ncyxij,kij->nyxck", blocks(imgs), B).reshape(G, 2, Ht, Wt, 12)
    i_t, p_t = tok[:, 0], tok[:, 1]
    num = (i_t * p_t).sum(-1)
    den = i_t.norm(dim=-1) * p_t.norm(dim=-1)
    sim = torch.where(den > 0, num / den.clamp_min(1e-300), torch.ones_like(num)).clamp(-1, 1)
    kdrop = int(drop * Ht * Wt + 0.5)
    idx = torch.topk(sim.view(G, -1), kdrop, dim=1).indices
    keep = torch.ones(G, Ht * Wt, dtype=torch.bool, device=dev).scatter_(1, idx, False)
    p_t = p_t * keep.view(G, Ht, Wt, 1)
    q = torch.stack([i_t, p_t], 1)                  # per-row 8-bit quantisation
    qmin = q.amin(dim=(3, 4), keepdim=True).float().double()
    qr = (q.amax(dim=(3, 4), keepdim=True) - q.amin(dim=(3, 4), keepdim=True)).float().double()
    lv = torch.round((q - qmin) * (255.0 / qr.clamp_min(1e-30))).clamp(0, 255)
    deq = qmin + lv * (qr / 255.0)
    deq[:, 1] = torch.where(keep.view(G, Ht, Wt, 1), deq[:, 1], deq[:, 0])   # concealment
    rec = torch.einsum("nyxck,kij->ncyixj", deq.view(G * 2, Ht, Wt, 3, 4), B)
    rec = rec.reshape(G * 2, 3, Ht * 8, Wt * 8)[:, :, :h, :w].clamp(0, 1)
    up = F.interpolate(rec, scale_factor=s, mode="bilinear", align_corners=False)
    up = up[:, :, :H, :W].clamp(0, 1).view(G, 2, 3, H, W).permute(0, 1, 3, 4, 2)
    out[:, 0] = 0.5 * prev_up + 0.5 * up[:, 0]
    out[:, 1:] = up[:, 1:2].to(torch.float32)
    return up[:, 1]


def timed(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


frames = torch.rand((G, 9, H, W, 3), device=dev)
out = torch.empty_like(frames)
prev = torch.rand((G, H, W, 3), device=dev, dtype=f64)
with torch.no_grad():
    lib_ms = timed(lambda: step(frames, prev, out))
bank = StreamBank(G, H, W, scales=(s,))
ours = lambda: bank.step({s: frames}, {s: out}, {s: list(range(G))}, {s: [0] * G},
                         drop_rate=drop)
ours()                                                     # prime the blend history
our_ms = timed(ours)
print(json.dumps({"G": G, "shape": "1080p, s=3, 10% drop, blend n=2",
                  "torch_f64_ms": round(lib_ms, 3), "fused_kernels_ms": round(our_ms, 3),
                  "speedup": round(lib_ms / our_ms, 2),
                  "frames_per_s": {"torch": round(G * 9 / lib_ms * 1e3),
                                   "fused": round(G * 9 / our_ms * 1e3)}}))
