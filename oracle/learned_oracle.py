"""ORACLE / TEST INFRASTRUCTURE ONLY -- parity UNPINNED.

torch fp32 CPU restatement of the learned-tokenizer plug-in
(``paper_2602_03529_b200/learned.py``), used by
``tests/`` as the checker for the tcgen05 kernels in ``csrc/learned.cu``.

Why unpinned: the reference package ships no learned tokenizer (
the paper's Cosmos-based model, is not in
``/root/reference``), so there is no reference output to pin against.  What
this oracle does pin is the *definition*: the same network, written with
``torch.nn.functional.conv3d`` (an independent formulation from the kernels'
tap-major implicit GEMM), with the same bf16 rounding points:

* inputs, weights and every stored activation are bf16 values; convolutions
  accumulate in fp32;
* epilogue order per layer: +bias, then SiLU (if any), then +residual, then
  round to bf16 (STORE); +bias, FSQ (FSQ head); +bias, clamp to [0, 1]
  (unpatchify);
* FSQ: bound(z) = tanh(z + atanh(offset/half_l)) * half_l - offset with
  half_l = (L-1)(1-1e-3)/2, offset = 0.5 for even L; code = round-half-even
  (bound) / (L // 2); index = mixed radix over (8,8,8,5,5,5) per 6-dim group
  (Mentzer et al., "Finite Scalar Quantization", 2023).

The GPU and this oracle differ only in fp32 summation order (and the fast
exp in SiLU), so stored bf16 activations agree to within one bf16 ulp and
FSQ indices agree except where a bound value sits on a rounding boundary.
Tolerances (north_star, BASELINE.json): FSQ index agreement >= 99.9 %,
reconstruction max |err| <= 1e-2 in bf16 and PSNR within 0.05 dB.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

from oracle import semstream_oracle as O

FSQ_LEVELS = (8, 8, 8, 5, 5, 5, 8, 8, 8, 5, 5, 5)
BASIS = (1, 8, 64, 512, 2560, 12800)


def bf(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16).to(torch.float32)


def patchify(frames: np.ndarray, s: int):
    """frames float32 [G][9][H][W][3] -> (pI [G][H'][W'][192], pP [G][H'][W'][1536]),
    bf16 values as float32.  Downscale = the bit-exact box filter
    (codec.py:202-214), pad = edge to the 8 grid (codec.py:99-105)."""
    fr = np.asarray(frames, dtype=np.float32)
    if s > 1:
        fr = O.downscale(fr, s)
    G, T, h, w, _ = fr.shape
    Ht, Wt = -(-h // 8), -(-w // 8)
    fr = np.pad(fr, ((0, 0), (0, 0), (0, Ht * 8 - h), (0, Wt * 8 - w), (0, 0)), mode="edge")
    t = torch.from_numpy(np.ascontiguousarray(fr))
    # [G][9][Ht][8][Wt][8][3] -> [G][Ht][Wt][9][8][8][3]
    t = t.reshape(G, T, Ht, 8, Wt, 8, 3).permute(0, 2, 4, 1, 3, 5, 6)
    pI = bf(t[:, :, :, 0].reshape(G, Ht, Wt, 192))
    pP = bf(t[:, :, :, 1:].reshape(G, Ht, Wt, 1536))
    return pI, pP, (h, w)


def conv233(x: torch.Tensor, W: np.ndarray, b: np.ndarray, act: bool = False,
            residual: torch.Tensor | None = None) -> torch.Tensor:
    """Causal (2,3,3) conv of x [G][2][H][W][C] -> [G][2][H][W][N] (bf16 values)."""
    G, T, H, Wd, Cin = x.shape
    N = W.shape[0]
    w = torch.from_numpy(np.ascontiguousarray(W)).reshape(N, 2, 3, 3, Cin).permute(0, 4, 1, 2, 3)
    xin = x.permute(0, 4, 1, 2, 3)                              # [G][C][T][H][W]
    xin = F.pad(xin, (1, 1, 1, 1, 1, 0))                        # W, H both sides; T causal
    y = F.conv3d(xin, w.contiguous()).permute(0, 2, 3, 4, 1)    # [G][T][H][W][N]
    y = y + torch.from_numpy(np.asarray(b, dtype=np.float32))
    if act:
        y = F.silu(y)
    if residual is not None:
        y = y + residual
    return bf(y)


def linear(x: torch.Tensor, W: np.ndarray, b: np.ndarray) -> torch.Tensor:
    return x @ torch.from_numpy(np.ascontiguousarray(W)).T + torch.from_numpy(
        np.asarray(b, dtype=np.float32))


def fsq(z: torch.Tensor):
    """z [..., 12] fp32 -> (codes float64 [..., 12], indices int64 [..., 2])."""
    codes, idx = [], [torch.zeros(z.shape[:-1], dtype=torch.int64) for _ in range(2)]
    for i, L in enumerate(FSQ_LEVELS):
        half_l32 = np.float32((L - 1) * (1.0 - 1e-3) * 0.5)
        offset32 = np.float32(0.5 if L % 2 == 0 else 0.0)
        shift = torch.tensor(np.float32(np.arctanh(float(offset32) / float(half_l32))))
        half_l = torch.tensor(half_l32)
        offset = torch.tensor(offset32)
        bnd = torch.tanh(z[..., i] + shift) * half_l - offset
        q = torch.round(bnd).to(torch.int64)
        hw = L // 2
        codes.append(q.to(torch.float64) / hw)
        idx[i // 6] += (q + hw) * BASIS[i % 6]
    return torch.stack(codes, -1), torch.stack(idx, -1)


def window_attention(qkv: torch.Tensor) -> torch.Tensor:
    """Causal spatio-temporal 8x8-window attention (sst_lt_attn): qkv
    [G][2][H][W][3D] bf16 values -> [G][2][H][W][D] bf16 values.  Keys: the
    valid tokens of the query's window in latent frames <= its own; scores
    scaled by 1/sqrt(64), P = exp(s - max) in fp32 rounded to bf16 (the
    tensor-core operand), O = (P V) / sum(P) with the fp32 sum."""
    G, T, H, W, C3 = qkv.shape
    D = C3 // 3
    nh = D // 64
    Hp, Wp = -(-H // 8) * 8, -(-W // 8) * 8
    x = F.pad(qkv, (0, 0, 0, Wp - W, 0, Hp - H))
    valid = torch.zeros((Hp, Wp), dtype=torch.bool)
    valid[:H, :W] = True
    # [G][T][wy][8][wx][8][3][nh][64] -> [G][wy][wx][3][nh][T*64][64]
    x = x.reshape(G, T, Hp // 8, 8, Wp // 8, 8, 3, nh, 64)
    x = x.permute(0, 2, 4, 6, 7, 1, 3, 5, 8).reshape(G, Hp // 8, Wp // 8, 3, nh, T * 64, 64)
    q, k, v = x[:, :, :, 0], x[:, :, :, 1], x[:, :, :, 2]
    scores = (q @ k.transpose(-1, -2)) * 0.125
    kv = valid.reshape(Hp // 8, 8, Wp // 8, 8).permute(0, 2, 1, 3).reshape(Hp // 8, Wp // 8, 64)
    kv = kv.repeat(1, 1, T)                                    # [wy][wx][T*64] key validity
    frame = torch.arange(T * 64) // 64
    causal = frame[None, :] <= frame[:, None]                  # [query][key]
    allow = causal[None, None] & kv[:, :, None, :]             # [wy][wx][q][k]
    scores = scores.masked_fill(~allow[None, :, :, None], float("-inf"))
    # softmax with the unnormalised probabilities rounded to bf16 before P.V
    # (the tensor-core operand) and the fp32 row sum applied afterwards
    mx = scores.amax(-1, keepdim=True)
    p = torch.exp(scores - torch.where(torch.isfinite(mx), mx, torch.zeros_like(mx)))
    l = p.sum(-1, keepdim=True)
    o = (bf(p) @ v) / torch.where(l > 0, l, torch.ones_like(l))   # [G][wy][wx][nh][T*64][64]
    o = o.reshape(G, Hp // 8, Wp // 8, nh, T, 8, 8, 64).permute(0, 4, 1, 5, 2, 6, 3, 7)
    o = o.reshape(G, T, Hp, Wp, D)[:, :, :H, :W]
    return bf(o)


def attention_block(h: torch.Tensor, Wm: dict, bm: dict, part: str) -> torch.Tensor:
    qkv = bf(linear(h, Wm[f"{part}_qkv"], bm[f"{part}_qkv"]))
    o = window_attention(qkv)
    return bf(linear(o, Wm[f"{part}_proj"], bm[f"{part}_proj"]) + h)


def encode(frames: np.ndarray, s: int, weights: dict, blocks: int):
    """-> (codes f64 [G][2][H'][W'][12], idx [G][2][H'][W'][2], (h, w), latent before FSQ)."""
    Wm, bm = weights["W"], weights["b"]
    pI, pP, hw = patchify(frames, s)
    h0 = bf(linear(pI, Wm["pe_i"], bm["pe_i"]))
    h1 = bf(linear(pP, Wm["pe_p"], bm["pe_p"]))
    h = torch.stack([h0, h1], 1)
    for i in range(blocks):
        u = conv233(h, Wm[f"enc{i}_c1"], bm[f"enc{i}_c1"], act=True)
        h = conv233(u, Wm[f"enc{i}_c2"], bm[f"enc{i}_c2"], residual=h)
    if "enc_qkv" in Wm:
        h = attention_block(h, Wm, bm, "enc")
    z = linear(h, Wm["head"], bm["head"])[..., :12]
    codes, idx = fsq(z)
    return codes.numpy(), idx.numpy(), hw, z


def dec_in(tokens: np.ndarray, mask: np.ndarray) -> torch.Tensor:
    """Snap to the FSQ grid and conceal masked P tokens with the I token."""
    tok = np.array(tokens, dtype=np.float64)
    m = np.asarray(mask).astype(bool)
    src = tok.copy()
    src_m = m.copy()
    lost = ~m[:, 1]
    src[:, 1][lost] = tok[:, 0][lost]
    src_m[:, 1][lost] = m[:, 0][lost]
    out = np.zeros(tok.shape[:-1] + (64,), np.float32)
    for i, L in enumerate(FSQ_LEVELS):
        hw = L // 2
        q = np.clip(np.rint(src[..., i] * hw), -hw, L - 1 - hw)
        out[..., i] = (q / hw).astype(np.float32)
    out[~src_m] = 0.0
    return bf(torch.from_numpy(out))


def decode(tokens: np.ndarray, mask: np.ndarray, hw, weights: dict, blocks: int) -> np.ndarray:
    """-> frames float32 [G][9][h][w][3]."""
    Wm, bm = weights["W"], weights["b"]
    x = dec_in(tokens, mask)
    h = conv233(x, Wm["dec_in"], bm["dec_in"], act=True)
    if "dec_qkv" in Wm:
        h = attention_block(h, Wm, bm, "dec")
    for i in range(blocks):
        u = conv233(h, Wm[f"dec{i}_c1"], bm[f"dec{i}_c1"], act=True)
        h = conv233(u, Wm[f"dec{i}_c2"], bm[f"dec{i}_c2"], residual=h)
    oi = linear(h[:, 0], Wm["out_i"], bm["out_i"]).clamp(0.0, 1.0)     # [G][Ht][Wt][192]
    op = linear(h[:, 1], Wm["out_p"], bm["out_p"]).clamp(0.0, 1.0)     # [G][Ht][Wt][1536]
    G, Ht, Wt, _ = oi.shape
    fi = oi.reshape(G, Ht, Wt, 1, 8, 8, 3)
    fp = op.reshape(G, Ht, Wt, 8, 8, 8, 3)
    f = torch.cat([fi, fp], 3)                               # [G][Ht][Wt][9][8][8][3]
    f = f.permute(0, 3, 1, 4, 2, 5, 6).reshape(G, 9, Ht * 8, Wt * 8, 3)
    h_, w_ = hw
    return np.ascontiguousarray(f[:, :, :h_, :w_].numpy())
