"""ORACLE / TEST INFRASTRUCTURE ONLY -- parity UNPINNED (no reference model).

Exact integer restatement (numpy int64) of the int8 learned tokenizer
(``paper_2602_03529_b200/learned_i8.py``), the checker
for the kind::i8 tcgen05 kernels in ``csrc/learned_i8.cu``.

The reference package ships no learned tokenizer (the paper's
Cosmos-based model, is not in ``/root/reference``), so the
network's *definition* is pinned here, not its weights: every operation is
integer arithmetic (int8 x int8 products summed in int64 / int32 -- exact in
any order), integer requantisation with arithmetic shifts, and table
lookups for the two non-linearities.  Nothing depends on summation order or
on a transcendental function's last ulp, so the GPU must agree BIT FOR BIT:
FSQ indices 100 %, decoded frames identical.  (The bf16 model's oracle,
``learned_oracle.py``, can only bound its agreement: fp32 summation order
differs between tensor cores and the CPU.)

Definitions (shared with the kernels; ``r(x, s) = (x + 2^(s-1)) >> s``,
arithmetic shift = floor):

* pixel -> int8: ``rint(float64(px) * 255) - 128`` of the bit-exact
  working-resolution frame (codec.py:202-214 downscale, codec.py:99-105 edge
  pad), patchified to I [H'][W'][192 -> 256 zero-padded] and P [H'][W'][1536]
  (optionally through an integer 3-D Haar front end, ``haar_front``);
* layer: ``acc = sum_k x[k] * W[n][k]`` (K order tap-major, channel-minor;
  (2,3,3) taps see latent frames t-1, t and a 3x3 neighbourhood, zero
  outside), ``y = clamp(r(acc + b[n], sh), -127, 127)``, then SiLU as a
  256-entry int8 table, then ``clamp(residual + y, -127, 127)``;
* attention (8x8 token windows x 2 latent frames, 128-dim heads, causal in
  time): ``S = Q K^T`` (int32), ``e = EXP[min((max - S) >> sh_s, 255)]``
  (uint8 table, EXP[0] = 255), ``l = sum e``, ``O = sum e V``,
  ``out = clamp(floor((2 O + l) / (2 l)), -127, 127)``;
* FSQ head: ``q_c = clamp((acc + b) >> sh_h, -L/2, L-1-L/2)`` for levels
  (8,8,8,5,5,5) x 2, code = q / (L/2) (float64), index = mixed radix of
  q + L/2;
* decoder input: received codes snapped back to q (codec-side 8-bit wire
  error << half a step), masked P tokens concealed by the co-located I token
  (codec.py:176-180 in latent space), ``x = 16 q``; the first decoder layer's
  (2,3,3) neighbourhood is gathered into 2 x 9 x 12 = 216 (+40 zero) channels
  so it runs as one K = 256 GEMM;
* pixels: ``clamp(r(acc + b, sh), 0, 255) / 255`` in float32.
"""

from __future__ import annotations

import numpy as np

from oracle import semstream_oracle as O

FSQ_LEVELS = (8, 8, 8, 5, 5, 5, 8, 8, 8, 5, 5, 5)
BASIS = (1, 8, 64, 512, 2560, 12800)
TAPS_233 = [(kt - 1, ky - 1, kx - 1) for kt in range(2) for ky in range(3) for kx in range(3)]
WIN = 8


def rshift_round(x: np.ndarray, sh: int) -> np.ndarray:
    x = np.asarray(x, dtype=np.int64)
    return (x + (1 << (sh - 1))) >> sh if sh > 0 else x


def requant(acc: np.ndarray, b: np.ndarray, sh: int, lut=None, residual=None) -> np.ndarray:
    y = np.clip(rshift_round(acc + np.asarray(b, np.int64), sh), -127, 127)
    if lut is not None:
        y = np.asarray(lut, np.int64)[y + 128]
    if residual is not None:
        y = np.clip(np.asarray(residual, np.int64) + y, -127, 127)
    return y.astype(np.int8)


def gemm(x: np.ndarray, W: np.ndarray) -> np.ndarray:
    """int8 [..., K] x int8 [N][K] -> int64 [..., N], exact (float64 BLAS on
    integers < 2^53 is exact in any order)."""
    xs = x.reshape(-1, x.shape[-1]).astype(np.float64)
    out = xs @ np.asarray(W, np.float64).T
    return out.astype(np.int64).reshape(x.shape[:-1] + (W.shape[0],))


def im2col233(x: np.ndarray) -> np.ndarray:
    """[G][T][H][W][C] -> [G][T][H][W][18 C] (tap-major, zero padding)."""
    G, T, H, W, C = x.shape
    xp = np.zeros((G, T + 1, H + 2, W + 2, C), dtype=x.dtype)
    xp[:, 1:, 1:H + 1, 1:W + 1] = x
    cols = [xp[:, 1 + dt:1 + dt + T, 1 + dy:1 + dy + H, 1 + dx:1 + dx + W]
            for dt, dy, dx in TAPS_233]
    return np.concatenate(cols, axis=-1)


def conv233(x, w, name, act=False, residual=None):
    acc = gemm(im2col233(x), w["W"][name])
    return requant(acc, w["b"][name], w["sh"][name], w["silu"] if act else None, residual)


def linear(x, w, name, act=False, residual=None):
    acc = gemm(x, w["W"][name])
    return requant(acc, w["b"][name], w["sh"][name], w["silu"] if act else None, residual)


def quantize_pixels(px: np.ndarray) -> np.ndarray:
    return (np.rint(np.asarray(px, np.float32).astype(np.float64) * 255.0) - 128.0).astype(np.int8)


def haar_step(x: np.ndarray, axis: int, m: int) -> np.ndarray:
    """One integer Haar analysis step on the first ``m`` entries of ``axis``:
    pairs (a, b) = (x[2j], x[2j+1]) -> lo = (a + b) >> 1 at j, hi = (a - b) >> 1
    at m/2 + j (floors; int8 in, int8 out: both stay in [-128, 127])."""
    x = np.moveaxis(np.asarray(x, np.int64), axis, 0).copy()
    a, b = x[0:m:2].copy(), x[1:m:2].copy()
    x[:m // 2] = (a + b) >> 1
    x[m // 2:m] = (a - b) >> 1
    return np.moveaxis(x, 0, axis)


def haar3(x: np.ndarray, axes) -> np.ndarray:
    """Three dyadic levels (8 -> 4 -> 2 -> 1 low band) of the separable Haar
    over ``axes`` (each of length 8), Mallat layout: at each level the low
    band's region [0:m] along every axis is transformed, axes in the given
    order (for the spatial pair: horizontal first, then vertical)."""
    for m in (8, 4, 2):
        sl = [slice(None)] * x.ndim
        for ax in axes:
            sl[ax] = slice(0, m)
        sub = x[tuple(sl)]
        for ax in axes:
            sub = haar_step(sub, ax, m)
        x = np.asarray(x, np.int64).copy()
        x[tuple(sl)] = sub
    return x


def haar_front(q: np.ndarray) -> np.ndarray:
    """Integer 3-D Haar wavelet front end (Cosmos' first stage),
    applied to the quantised, patch-split pixels q int [G][Ht][Wt][9][8][8][3]
    (frame, row, column, channel): the eight P frames get three temporal
    levels (the I frame is the causal first frame and is transformed only in
    space), then every frame slot three spatial levels (rows' horizontal pairs,
    then columns').  Same coefficient layout as the pixels it replaces."""
    q = np.asarray(q, np.int64).copy()
    q[:, :, :, 1:] = haar3(q[:, :, :, 1:], (3,))
    return haar3(q, (5, 4))


def patchify(frames: np.ndarray, s: int, front: str = "patch"):
    """frames float32 [G][9][H][W][3] -> pI int8 [G][1][H'][W'][256] (192 used),
    pP int8 [G][1][H'][W'][1536].  ``front="haar"`` inserts ``haar_front``."""
    fr = np.asarray(frames, dtype=np.float32)
    if s > 1:
        fr = O.downscale(fr, s)
    G, T, h, w, _ = fr.shape
    Ht, Wt = -(-h // 8), -(-w // 8)
    fr = np.pad(fr, ((0, 0), (0, 0), (0, Ht * 8 - h), (0, Wt * 8 - w), (0, 0)), mode="edge")
    q = quantize_pixels(fr).reshape(G, T, Ht, 8, Wt, 8, 3).transpose(0, 2, 4, 1, 3, 5, 6)
    if front == "haar":
        q = haar_front(q).astype(np.int8)
    elif front != "patch":
        raise ValueError(f"front must be 'patch' or 'haar', got {front!r}")
    pI = np.zeros((G, 1, Ht, Wt, 256), np.int8)
    pI[:, 0, :, :, :192] = q[:, :, :, 0].reshape(G, Ht, Wt, 192)
    pP = q[:, :, :, 1:].reshape(G, 1, Ht, Wt, 1536)
    return pI, pP, (h, w)


def _window_tokens(x: np.ndarray, Ht: int, Wt: int):
    """[G][2][Ht][Wt][C] -> ([G][wy][wx][128][C] zero-padded, valid [wy][wx][128])."""
    G, T, _, _, C = x.shape
    wy, wx = -(-Ht // WIN), -(-Wt // WIN)
    xp = np.zeros((G, T, wy * WIN, wx * WIN, C), x.dtype)
    xp[:, :, :Ht, :Wt] = x
    v = np.zeros((T, wy * WIN, wx * WIN), bool)
    v[:, :Ht, :Wt] = True
    xw = xp.reshape(G, T, wy, WIN, wx, WIN, C).transpose(0, 2, 4, 1, 3, 5, 6)
    vw = v.reshape(T, wy, WIN, wx, WIN).transpose(1, 3, 0, 2, 4)
    return xw.reshape(G, wy, wx, T * WIN * WIN, C), vw.reshape(wy, wx, T * WIN * WIN)


def attention_core(qkv: np.ndarray, D: int, hd: int, sh_s: int, exp_lut) -> np.ndarray:
    """qkv int8 [G][2][Ht][Wt][3D] -> out int8 [G][2][Ht][Wt][D]."""
    G, T, Ht, Wt, _ = qkv.shape
    xw, vw = _window_tokens(qkv, Ht, Wt)                 # [G][wy][wx][128][3D]
    n = xw.shape[3]
    frame = np.arange(n) // (WIN * WIN)
    causal = frame[None, :] <= frame[:, None]            # [q][k]
    allowed = causal[None, None] & vw[:, :, None, :]      # [wy][wx][q][k]
    lut = np.asarray(exp_lut, np.int64)
    outw = np.zeros(xw.shape[:4] + (D,), np.int64)
    for h in range(D // hd):
        q = xw[..., h * hd:(h + 1) * hd].astype(np.int64)
        k = xw[..., D + h * hd:D + (h + 1) * hd].astype(np.int64)
        v = xw[..., 2 * D + h * hd:2 * D + (h + 1) * hd].astype(np.int64)
        S = np.einsum("gyxqd,gyxkd->gyxqk", q.astype(np.float64), k.astype(np.float64)
                      ).astype(np.int64)
        Sm = np.where(allowed[None], S, np.iinfo(np.int64).min)
        m = Sm.max(axis=-1, keepdims=True)
        d = np.minimum((m - np.where(allowed[None], S, m)) >> sh_s, 255)
        e = np.where(allowed[None], lut[d], 0)
        l_ = e.sum(axis=-1, keepdims=True)
        Ov = np.einsum("gyxqk,gyxkd->gyxqd", e.astype(np.float64), v.astype(np.float64)
                       ).astype(np.int64)
        outw[..., h * hd:(h + 1) * hd] = np.clip((2 * Ov + l_) // (2 * l_), -127, 127)
    wy, wx = vw.shape[:2]
    out = outw.reshape(G, wy, wx, T, WIN, WIN, D).transpose(0, 3, 1, 4, 2, 5, 6)
    out = out.reshape(G, T, wy * WIN, wx * WIN, D)[:, :, :Ht, :Wt]
    return out.astype(np.int8)


def attention_core_global(qkv: np.ndarray, D: int, hd: int, sh_s: int, exp_lut) -> np.ndarray:
    """Global causal attention: a query of latent frame t attends every token
    of frames <= t (all H' x W' positions, no windows); same integer softmax."""
    G, T, Ht, Wt, _ = qkv.shape
    n = Ht * Wt
    x = qkv.reshape(G, T * n, 3 * D)
    frame = np.arange(T * n) // n
    allowed = frame[None, :] <= frame[:, None]                     # [q][k]
    lut = np.asarray(exp_lut, np.int64)
    out = np.zeros((G, T * n, D), np.int64)
    for g in range(G):
        for h in range(D // hd):
            q = x[g, :, h * hd:(h + 1) * hd].astype(np.float64)
            k = x[g, :, D + h * hd:D + (h + 1) * hd].astype(np.float64)
            v = x[g, :, 2 * D + h * hd:2 * D + (h + 1) * hd].astype(np.float64)
            S = (q @ k.T).astype(np.int64)
            m = np.where(allowed, S, np.iinfo(np.int64).min).max(axis=-1, keepdims=True)
            d = np.minimum((m - np.where(allowed, S, m)) >> sh_s, 255)
            e = np.where(allowed, lut[d], 0)
            l_ = e.sum(axis=-1, keepdims=True)
            Ov = (e.astype(np.float64) @ v).astype(np.int64)
            out[g, :, h * hd:(h + 1) * hd] = np.clip((2 * Ov + l_) // (2 * l_), -127, 127)
    return out.reshape(G, T, Ht, Wt, D).astype(np.int8)


def attention_block(h: np.ndarray, w: dict, part: str) -> np.ndarray:
    D = h.shape[-1]
    qkv = linear(h, w, f"{part}_qkv")
    core = attention_core_global if w.get("attn_scope") == "global" else attention_core
    o = core(qkv, D, w["head_dim"], w["attn_shift"], w["exp"])
    return linear(o, w, f"{part}_proj", residual=h)


def fsq(acc: np.ndarray, b: np.ndarray, sh: int):
    """int64 head accumulators [..., 16] -> (codes f64 [..., 12], idx i32 [..., 2])."""
    z = (acc[..., :12] + np.asarray(b, np.int64)[:12]) >> sh
    L = np.array(FSQ_LEVELS)
    hw = L // 2
    q = np.clip(z, -hw, L - 1 - hw)
    codes = q.astype(np.float64) / hw.astype(np.float64)
    digits = (q + hw) * np.array(BASIS * 2)
    idx = np.stack([digits[..., :6].sum(-1), digits[..., 6:].sum(-1)], -1).astype(np.int32)
    return codes, idx


def encode(frames: np.ndarray, s: int, w: dict):
    """-> (codes f64 [G][2][H'][W'][12], idx i32 [G][2][H'][W'][2], (h, w))."""
    pI, pP, hw = patchify(frames, s, w.get("front", "patch"))
    h0 = linear(pI, w, "pe_i")
    h1 = linear(pP, w, "pe_p")
    h = np.concatenate([h0, h1], axis=1)
    for i in range(w["blocks"]):
        u = conv233(h, w, f"enc{i}_c1", act=True)
        h = conv233(u, w, f"enc{i}_c2", residual=h)
    if w["attn"]:
        h = attention_block(h, w, "enc")
    codes, idx = fsq(gemm(h, w["W"]["head"]), w["b"]["head"], w["sh"]["head"])
    return codes, idx, hw


def snap_codes(tokens: np.ndarray, mask: np.ndarray) -> np.ndarray:
    """Received f64 codes [G][2][H'][W'][12] + mask -> int8 16 q, concealed."""
    tok = np.asarray(tokens, np.float64).copy()
    m = np.asarray(mask).astype(bool).copy()
    conceal = ~m[:, 1]
    tok[:, 1][conceal] = tok[:, 0][conceal]
    m[:, 1][conceal] = m[:, 0][conceal]
    L = np.array(FSQ_LEVELS)
    hw = L // 2
    q = np.clip(np.rint(tok * hw), -hw, L - 1 - hw).astype(np.int64)
    q = np.where(m[..., None], q, 0)
    return (16 * q).astype(np.int8)


def dec_input(codes_q: np.ndarray) -> np.ndarray:
    """int8 [G][2][H'][W'][12] -> int8 [G][2][H'][W'][256]: the (2,3,3)
    neighbourhood gathered tap-major (216 channels), zero-padded."""
    G, T, Ht, Wt, _ = codes_q.shape
    cols = im2col233(codes_q)                         # [G][2][Ht][Wt][216]
    out = np.zeros((G, T, Ht, Wt, 256), np.int8)
    out[..., :216] = cols
    return out


def decode_inputs(x: np.ndarray, hw, w: dict) -> np.ndarray:
    """Decoder from its gathered int8 input -> frames f32 [G][9][h][w][3]."""
    h = linear(x, w, "dec_in", act=True)
    if w["attn"]:
        h = attention_block(h, w, "dec")
    for i in range(w["blocks"]):
        u = conv233(h, w, f"dec{i}_c1", act=True)
        h = conv233(u, w, f"dec{i}_c2", residual=h)
    G, _, Ht, Wt, _ = h.shape
    hh, ww = hw
    pix_i = gemm(h[:, 0], w["W"]["out_i"])           # [G][Ht][Wt][192]
    pix_p = gemm(h[:, 1], w["W"]["out_p"])           # [G][Ht][Wt][1536]
    frames = np.zeros((G, 9, Ht * 8, Wt * 8, 3), np.float32)

    def px(acc, name):
        q = np.clip(rshift_round(acc + np.asarray(w["b"][name], np.int64), w["sh"][name]), 0, 255)
        return q.astype(np.float32) / np.float32(255.0)

    fi = px(pix_i, "out_i").reshape(G, Ht, Wt, 8, 8, 3).transpose(0, 1, 3, 2, 4, 5)
    frames[:, 0] = fi.reshape(G, Ht * 8, Wt * 8, 3)
    fp = px(pix_p, "out_p").reshape(G, Ht, Wt, 8, 8, 8, 3).transpose(0, 3, 1, 4, 2, 5, 6)
    frames[:, 1:] = fp.reshape(G, 8, Ht * 8, Wt * 8, 3)
    return frames[:, :, :hh, :ww]


def decode(tokens: np.ndarray, mask: np.ndarray, hw, w: dict) -> np.ndarray:
    return decode_inputs(dec_input(snap_codes(tokens, mask)), hw, w)
