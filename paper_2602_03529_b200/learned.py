"""Learned tokenizer plug-in: a causal spatio-temporal
convolutional tokenizer with finite-scalar quantisation (FSQ), run on the
B200's tensor cores and plugged in at the reference's tokenizer hook.

The reference (`semstream`) ships no learned model: its tokenizer is a fixed
8x8 block-DCT proxy "behind the same interface a learned model would use"
(pkg/README.md:3-7).  The paper's codec is a Cosmos-style
tokenizer: causal spatio-temporal blocks, 8x spatial and 8x
temporal compression, FSQ latents.  This module is that shape of model behind
the reference's plug-in contract (session.py:57-61):

    encode(GoP, CodecConfig) -> (TokenMatrix I, TokenMatrix P)
    decode(TokenMatrix I, TokenMatrix P, CodecConfig) -> GoP

Geometry (identical to the proxy so packetisation, intelligent dropping and
reassembly are reused unchanged):

  * a 9-frame GoP at working resolution h x w is edge-padded to the 8x8 grid
    (codec.py:99-105) and patchified: latent frame t=0 (I) embeds frame 0's
    8x8x3 patch, latent frame t=1 (P) embeds frames 1..8's 8x8x8x3 patch;
  * encoder: patch embeddings -> D channels, `blocks` causal residual blocks
    h += conv(SiLU(conv(h))) with (2,3,3) kernels that see t and t-1 only,
    a causal spatio-temporal attention block h += proj(attn(qkv(h))) (8x8
    token windows, 64-dim heads, frame t attends to frames <= t), then a 1x1
    head to 12 channels and FSQ (two groups of levels
    (8,8,8,5,5,5), 64000 codes each).  The 12 FSQ code values are the
    TokenMatrix channels (codec.py:32 fixes C = 12) and travel through the
    reference's 8-bit row quantiser; the decoder snaps them back onto the FSQ
    grid, which is lossless because the quantiser error (<= range/510) is far
    below half an FSQ step;
  * decoder: masked P tokens take the co-located I token's codes (the
    proxy's concealment rule, codec.py:176-180, in latent space), a (2,3,3)
    conv lifts 12 -> D channels, an attention block, `blocks` residual
    blocks, then 1x1 unpatchify
    convs write frame 0 (from t=0) and frames 1..8 (from t=1), clamped to
    [0, 1] and cropped to the working frame.

Every convolution is one `sst_lt_conv` launch: an implicit GEMM on tcgen05
(bf16 operands, fp32 accumulation in TMEM, TMA-fed, fused epilogue).
Weights are seeded random-init (there is no checkpoint; BASELINE.json
configs[0] "random-init weights").  Parity is against the torch fp32
restatement in oracle/learned_oracle.py (unpinned: no reference model).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .codec import CodecConfig, TokenMatrix, token_grid_shape
from .pipeline import CHANNELS, GopCodec, check_gop_tensor
from .video import GOP_SIZE, Frame, GoP

FSQ_LEVELS = (8, 8, 8, 5, 5, 5, 8, 8, 8, 5, 5, 5)
FSQ_CHANNELS = len(FSQ_LEVELS)      # = CodecConfig.channels (codec.py:32)
DEC_IN_CHANNELS = 64                # FSQ codes zero-padded to one 128-byte K block
PATCH_I = 8 * 8 * 3
PATCH_P = 8 * 8 * 8 * 3

# (dt, dy, dx) of the causal (2,3,3) kernel, in K order (kt, ky, kx)
TAPS_233 = [(kt - 1, ky - 1, kx - 1) for kt in range(2) for ky in range(3) for kx in range(3)]


@dataclass(frozen=True)
class LearnedConfig:
    dim: int = 256          # latent channels D (multiple of 128)
    blocks: int = 2         # residual blocks in the encoder and in the decoder
    seed: int = 0
    attn: bool = True       # one causal spatio-temporal window-attention block per side

    def __post_init__(self):
        if self.dim <= 0 or self.dim % 128:
            raise ValueError(f"dim must be a positive multiple of 128, got {self.dim}")
        if not 0 <= self.blocks <= 8:
            raise ValueError(f"blocks must be in [0, 8], got {self.blocks}")


def _bf16_round(a: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(
        torch.bfloat16).to(torch.float32).numpy()


def make_weights(cfg: LearnedConfig) -> dict:
    """Seeded random-init weights as float32 arrays holding bf16 values.

    Layout: W[name] is [N][K] with K ordered (tap, input channel), the GEMM
    "B" operand of the implicit convolution; b[name] is [N] float32.
    """
    rng = np.random.default_rng(cfg.seed)
    D = cfg.dim

    def normal(n, k, std):
        return _bf16_round(rng.standard_normal((n, k)).astype(np.float32) * np.float32(std))

    W, b = {}, {}
    W["pe_i"] = normal(D, PATCH_I, 1.0 / np.sqrt(PATCH_I))
    W["pe_p"] = normal(D, PATCH_P, 1.0 / np.sqrt(PATCH_P))
    b["pe_i"] = _bf16_round(rng.standard_normal(D).astype(np.float32) * 0.1)
    b["pe_p"] = _bf16_round(rng.standard_normal(D).astype(np.float32) * 0.1)
    K3 = len(TAPS_233) * D
    for part in ("enc", "dec"):
        for i in range(cfg.blocks):
            W[f"{part}{i}_c1"] = normal(D, K3, np.sqrt(2.0 / K3))
            W[f"{part}{i}_c2"] = normal(D, K3, 0.3 / np.sqrt(K3))
            b[f"{part}{i}_c1"] = np.zeros(D, np.float32)
            b[f"{part}{i}_c2"] = np.zeros(D, np.float32)
    head = np.zeros((16, D), np.float32)
    head[:FSQ_CHANNELS] = normal(FSQ_CHANNELS, D, 1.5 / np.sqrt(D))
    W["head"] = head
    b["head"] = np.zeros(16, np.float32)
    # decoder input conv: only the 12 code channels of each tap carry weight
    w_in = np.zeros((D, len(TAPS_233), DEC_IN_CHANNELS), np.float32)
    w_in[:, :, :FSQ_CHANNELS] = normal(D, len(TAPS_233) * FSQ_CHANNELS,
                                       np.sqrt(2.0 / (len(TAPS_233) * FSQ_CHANNELS))).reshape(
        D, len(TAPS_233), FSQ_CHANNELS)
    W["dec_in"] = w_in.reshape(D, -1)
    b["dec_in"] = np.zeros(D, np.float32)
    W["out_i"] = normal(PATCH_I, D, 0.25 / np.sqrt(D))
    W["out_p"] = normal(PATCH_P, D, 0.25 / np.sqrt(D))
    b["out_i"] = np.full(PATCH_I, 0.5, np.float32)
    b["out_p"] = np.full(PATCH_P, 0.5, np.float32)
    if cfg.attn:     # drawn last: the weights above do not depend on cfg.attn
        for part in ("enc", "dec"):
            W[f"{part}_qkv"] = normal(3 * D, D, 1.0 / np.sqrt(D))
            b[f"{part}_qkv"] = np.zeros(3 * D, np.float32)
            W[f"{part}_proj"] = normal(D, D, 0.5 / np.sqrt(D))
            b[f"{part}_proj"] = np.zeros(D, np.float32)
    return {"W": W, "b": b}


def _taps_array(taps):
    arr = ((C.c_int32 * 3) * 27)()
    for i, (dt, dy, dx) in enumerate(taps):
        arr[i][0], arr[i][1], arr[i][2] = dt, dy, dx
    return arr


class LearnedTokenizer:
    """Device-resident learned tokenizer (weights bf16 on the GPU)."""

    def __init__(self, cfg: LearnedConfig | None = None, weights: dict | None = None):
        self.cfg = cfg or LearnedConfig()
        dev = _dev.device()
        host = weights if weights is not None else make_weights(self.cfg)
        self.host_weights = host
        self.W = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev).to(torch.bfloat16)
                  for k, v in host["W"].items()}
        self.b = {k: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).to(dev)
                  for k, v in host["b"].items()}
        self.launches = 0

    # ---- one layer ----------------------------------------------------------
    def _conv(self, name, x, in_shape, out_grid, taps, t_lo, t_cnt, epi, *, act=0,
              residual=None, out=None, out_T=2, codes=None, idx=None, mask=None, frames=None,
              hw=(0, 0), frame_base=0):
        G, T_in, H_in, W_in, C_in = in_shape
        Ht, Wt = out_grid
        W = self.W[name]
        d = _lib.SstConvDesc()
        d.in_ = x.data_ptr()
        d.in_C, d.in_W, d.in_H, d.in_T = C_in, W_in, H_in, T_in
        d.G, d.Ht, d.Wt, d.t_lo, d.t_cnt = G, Ht, Wt, t_lo, t_cnt
        d.n_taps = len(taps)
        d.taps = _taps_array(taps)
        d.weight = W.data_ptr()
        d.N, d.K = W.shape
        d.bias = self.b[name].data_ptr()
        d.epi, d.act = epi, act
        d.residual = residual.data_ptr() if residual is not None else None
        d.out = out.data_ptr() if out is not None else None
        d.out_T = out_T
        d.codes = codes.data_ptr() if codes is not None else None
        d.idx = idx.data_ptr() if idx is not None else None
        d.mask = mask.data_ptr() if mask is not None else None
        d.frames = frames.data_ptr() if frames is not None else None
        d.h, d.w = hw
        d.frame_base = frame_base
        _lib.call("sst_lt_conv", C.byref(d), _dev.stream())
        self.launches += 1

    def _blocks(self, part, h, u, G, Ht, Wt):
        D = self.cfg.dim
        shape = (G, 2, Ht, Wt, D)
        for i in range(self.cfg.blocks):
            self._conv(f"{part}{i}_c1", h, shape, (Ht, Wt), TAPS_233, 0, 2, _lib.LT_EPI_STORE,
                       act=1, out=u)
            self._conv(f"{part}{i}_c2", u, shape, (Ht, Wt), TAPS_233, 0, 2, _lib.LT_EPI_STORE,
                       residual=h, out=h)

    def _attention(self, part, h, G, Ht, Wt):
        """h += proj(WindowAttention(qkv(h))): the qkv projection and the
        8x8-window causal attention run in one persistent, warp-specialised
        tcgen05 kernel (sst_lt_attn_fused; SST_LT_ATTN=fused: one CTA per
        (window, head); SST_LT_ATTN=unfused: a 1x1 GEMM writing qkv, then
        sst_lt_attn), proj is a tcgen05 1x1 GEMM with the residual add."""
        if not self.cfg.attn:
            return
        D = self.cfg.dim
        shape = (G, 2, Ht, Wt, D)
        o = torch.empty_like(h)
        if os.environ.get("SST_LT_ATTN") != "unfused":
            # qkv projection inside the attention kernel (no qkv tensor)
            _lib.call("sst_lt_attn_fused", h.data_ptr(), self.W[f"{part}_qkv"].data_ptr(),
                      self.b[f"{part}_qkv"].data_ptr(), G, Ht, Wt, D, o.data_ptr(), _dev.stream())
            self.launches += 1
        else:
            qkv = torch.empty((G, 2, Ht, Wt, 3 * D), dtype=torch.bfloat16, device=h.device)
            self._conv(f"{part}_qkv", h, shape, (Ht, Wt), [(0, 0, 0)], 0, 2, _lib.LT_EPI_STORE,
                       out=qkv)
            _lib.call("sst_lt_attn", qkv.data_ptr(), G, Ht, Wt, D, o.data_ptr(), _dev.stream())
            self.launches += 1
        self._conv(f"{part}_proj", o, shape, (Ht, Wt), [(0, 0, 0)], 0, 2, _lib.LT_EPI_STORE,
                   residual=h, out=h)

    # ---- encoder ------------------------------------------------------------
    def encode_frames(self, frames: torch.Tensor, s: int = 1, codes: torch.Tensor | None = None,
                      mask: torch.Tensor | None = None, idx: torch.Tensor | None = None):
        """frames: float32 [G][9][H][W][3] on the GPU (full resolution when
        s in {2,3}: the box downscale is fused into the patchify pass).
        Returns (codes f64 [G][2][H'][W'][12], idx i32 [G][2][H'][W'][2],
        mask u8 [G][2][H'][W'], (h, w)); codes / mask / idx may be passed in
        (contiguous, G leading) to be written in place."""
        if frames.dtype != torch.float32 or frames.dim() != 5 or frames.shape[1] != GOP_SIZE \
                or frames.shape[4] != 3:
            raise ValueError("frames must be float32 [G][9][H][W][3]")
        frames = frames.contiguous()
        G, _, H, Wd, _ = frames.shape
        h, w = -(-H // s), -(-Wd // s)
        Ht, Wt = token_grid_shape(h, w)
        D = self.cfg.dim
        dev = frames.device
        pI = torch.empty((G, 1, Ht, Wt, PATCH_I), dtype=torch.bfloat16, device=dev)
        pP = torch.empty((G, 1, Ht, Wt, PATCH_P), dtype=torch.bfloat16, device=dev)
        st = _dev.stream()
        _lib.call("sst_lt_patchify", frames.data_ptr(), G, H, Wd, s, pI.data_ptr(),
                  pP.data_ptr(), st)
        self.launches += 1
        hbuf = torch.empty((G, 2, Ht, Wt, D), dtype=torch.bfloat16, device=dev)
        ubuf = torch.empty_like(hbuf)
        self._conv("pe_i", pI, (G, 1, Ht, Wt, PATCH_I), (Ht, Wt), [(0, 0, 0)], 0, 1,
                   _lib.LT_EPI_STORE, out=hbuf)
        self._conv("pe_p", pP, (G, 1, Ht, Wt, PATCH_P), (Ht, Wt), [(-1, 0, 0)], 1, 1,
                   _lib.LT_EPI_STORE, out=hbuf)
        self._blocks("enc", hbuf, ubuf, G, Ht, Wt)
        self._attention("enc", hbuf, G, Ht, Wt)
        if codes is None:
            codes = torch.zeros((G, 2, Ht, Wt, FSQ_CHANNELS), dtype=torch.float64, device=dev)
        if idx is None:
            idx = torch.zeros((G, 2, Ht, Wt, 2), dtype=torch.int32, device=dev)
        if mask is None:
            mask = torch.zeros((G, 2, Ht, Wt), dtype=torch.uint8, device=dev)
        for t_, shp in ((codes, (G, 2, Ht, Wt, FSQ_CHANNELS)), (idx, (G, 2, Ht, Wt, 2)),
                        (mask, (G, 2, Ht, Wt))):
            if tuple(t_.shape) != shp or not t_.is_contiguous():
                raise ValueError(f"output buffer must be a contiguous {shp} tensor")
        self._conv("head", hbuf, (G, 2, Ht, Wt, D), (Ht, Wt), [(0, 0, 0)], 0, 2,
                   _lib.LT_EPI_FSQ, codes=codes, idx=idx, mask=mask)
        return codes, idx, mask, (h, w)

    # ---- decoder ------------------------------------------------------------
    def decode_tokens(self, tokens: torch.Tensor, mask: torch.Tensor, hw,
                      frames: torch.Tensor | None = None) -> torch.Tensor:
        """tokens: float64 [G][2][H'][W'][12] (received, possibly 8-bit
        requantised codes; masked = 0), mask u8 [G][2][H'][W'].  Returns the
        working-resolution frames float32 [G][9][h][w][3]."""
        if tokens.dtype != torch.float64 or tokens.dim() != 5 or tokens.shape[1] != 2 \
                or tokens.shape[4] != FSQ_CHANNELS:
            raise ValueError("tokens must be float64 [G][2][H'][W'][12]")
        tokens = tokens.contiguous()
        mask = mask.to(torch.uint8).contiguous()
        G, _, Ht, Wt, _ = tokens.shape
        h, w = hw
        if not (0 < h <= Ht * 8 and 0 < w <= Wt * 8):
            raise ValueError(f"frame shape {hw} does not fit a {Ht}x{Wt} token grid")
        dev = tokens.device
        x = torch.empty((G, 2, Ht, Wt, DEC_IN_CHANNELS), dtype=torch.bfloat16, device=dev)
        _lib.call("sst_lt_dec_in", tokens.data_ptr(), mask.data_ptr(), G, Ht, Wt, x.data_ptr(),
                  _dev.stream())
        self.launches += 1
        return self.decode_inputs(x, hw, frames)

    def decode_inputs(self, x: torch.Tensor, hw, frames: torch.Tensor | None = None
                      ) -> torch.Tensor:
        """Decoder from its prepared input (bf16 [G][2][H'][W'][64]: snapped,
        concealed FSQ codes, e.g. sst_lt_unpack_dec_in straight from packets)."""
        G, _, Ht, Wt, _ = x.shape
        h, w = hw
        D = self.cfg.dim
        dev = x.device
        hbuf = torch.empty((G, 2, Ht, Wt, D), dtype=torch.bfloat16, device=dev)
        ubuf = torch.empty_like(hbuf)
        self._conv("dec_in", x, (G, 2, Ht, Wt, DEC_IN_CHANNELS), (Ht, Wt), TAPS_233, 0, 2,
                   _lib.LT_EPI_STORE, act=1, out=hbuf)
        self._attention("dec", hbuf, G, Ht, Wt)
        self._blocks("dec", hbuf, ubuf, G, Ht, Wt)
        if frames is None:
            frames = torch.empty((G, GOP_SIZE, h, w, 3), dtype=torch.float32, device=dev)
        elif tuple(frames.shape) != (G, GOP_SIZE, h, w, 3) or not frames.is_contiguous():
            raise ValueError("frames buffer must be a contiguous [G][9][h][w][3] tensor")
        self._conv("out_i", hbuf, (G, 2, Ht, Wt, D), (Ht, Wt), [(0, 0, 0)], 0, 1,
                   _lib.LT_EPI_PIXELS, frames=frames, hw=(h, w), frame_base=0)
        self._conv("out_p", hbuf, (G, 2, Ht, Wt, D), (Ht, Wt), [(0, 0, 0)], 1, 1,
                   _lib.LT_EPI_PIXELS, frames=frames, hw=(h, w), frame_base=1)
        return frames

    def flops_per_gop(self, Ht: int, Wt: int) -> int:
        """Tensor-core flops of one GoP (2 latent frames of Ht x Wt tokens),
        counting the padded GEMM shapes the kernels actually issue."""
        D, n = self.cfg.dim, Ht * Wt
        k3 = len(TAPS_233) * D
        enc = n * 2 * D * (PATCH_I + PATCH_P) + 2 * n * 2 * (2 * self.cfg.blocks * k3 * D) \
            + 2 * n * 2 * D * 16
        dec = 2 * n * 2 * len(TAPS_233) * DEC_IN_CHANNELS * D \
            + 2 * n * 2 * (2 * self.cfg.blocks * k3 * D) + n * 2 * D * (PATCH_I + PATCH_P)
        attn = 2 * (2 * n * 2 * D * 4 * D) if self.cfg.attn else 0   # qkv + proj, both sides
        return enc + dec + attn


# ---- the reference's plug-in contract (session.py:57-61) -------

class LearnedPlugin:
    """(encode, decode) pair for SessionConfig.tokenizer_encode/_decode.

    The plug-in receives the already downscaled working GoP
    (session.py:139-140), so the patchify runs at s = 1.
    """

    def __init__(self, cfg: LearnedConfig | None = None):
        self.model = LearnedTokenizer(cfg)

    def encode(self, gop: GoP, cfg: CodecConfig):
        frames = np.stack([f.samples for f in gop.frames])[None]
        codes, _, mask, (h, w) = self.model.encode_frames(_dev.h2d(frames, np.float32), 1)
        vals = _dev.d2h(codes)[0]
        m = _dev.d2h(mask)[0].astype(bool)
        return (TokenMatrix("I", vals[0], m[0], gop_id=gop.gop_id, frame_shape=(h, w)),
                TokenMatrix("P", vals[1], m[1], gop_id=gop.gop_id, frame_shape=(h, w)))

    def decode(self, i_tokens: TokenMatrix, p_tokens: TokenMatrix, cfg: CodecConfig) -> GoP:
        if i_tokens.values.shape != p_tokens.values.shape:
            raise ValueError("I and P token matrices differ in shape")
        if i_tokens.values.shape[2] != FSQ_CHANNELS:
            raise ValueError(f"learned tokenizer expects {FSQ_CHANNELS} channels")
        h, w = i_tokens.frame_shape
        tok = np.stack([i_tokens.values, p_tokens.values])[None]
        mask = np.stack([i_tokens.mask, p_tokens.mask])[None].astype(np.uint8)
        frames = _dev.d2h(self.model.decode_tokens(_dev.h2d(tok, np.float64),
                                                   _dev.h2d(mask, np.uint8), (h, w)))[0]
        out = tuple(Frame(frames[t], timestamp_index=t) for t in range(GOP_SIZE))
        return GoP(gop_id=i_tokens.gop_id, frames=out)


# ---- the batched device pipeline with the learned tokenizer ------------------

class LearnedGopCodec(GopCodec):
    """``pipeline.GopCodec`` with the learned tokenizer in place of the DCT
    proxy: the sender, transport and receiver stages are the reference's
    (session.py:134-170, 323-348) and reuse the proxy path's kernels:

      encode      learned encoder + FSQ (tcgen05) -> tokens [G][2][H'][W'][12]
      similarity  sst_similarity on the FSQ codes (selection.py:33-52)
      K2 / K3     intelligent drop + 8-bit packetisation with CRC (unchanged)
      K4          sst_parse + sst_lt_unpack_dec_in (first-wins routing; tokens
                  dequantised from the winning packets, concealed and snapped
                  straight into the first decoder conv's bf16 input)
      decode      mask-aware learned decoder (tcgen05), 9 distinct frames
      K5          sst_upscale (bilinear x s, crop) + sst_blend (Eq. 2)
    """

    def __init__(self, g_max: int, H: int, W: int, s: int, blend_n: int = 2,
                 model: LearnedTokenizer | None = None, cfg: LearnedConfig | None = None):
        super().__init__(g_max, H, W, s, blend_n)
        self.model = model if model is not None else LearnedTokenizer(cfg)
        dev = self.tok.device
        self.idx = torch.empty((g_max, 2, self.Ht, self.Wt, 2), dtype=torch.int32, device=dev)
        self.rx_tok = torch.empty_like(self.tok)
        self.rx_mask = torch.empty_like(self.mask)
        self.dec_x = torch.empty((g_max, 2, self.Ht, self.Wt, DEC_IN_CHANNELS),
                                 dtype=torch.bfloat16, device=dev)
        # double-buffered decoded frames: step k decodes into parity k % 2 while
        # boundary blending reads the previous step's frames from the other
        self.frames9 = [torch.empty((g_max, GOP_SIZE, self.h, self.w, 3), dtype=torch.float32,
                                    device=dev) for _ in range(2)]
        # SstPrevDesc[g_max] per parity: slot j's previous GoP = slot j of the other buffer
        self.prev_desc = []
        for par in range(2):
            d = np.zeros(g_max, dtype=_lib.PREV_DTYPE)
            src = self.frames9[1 - par]
            d["p_img"] = src.data_ptr() + np.arange(g_max, dtype=np.uint64) * np.uint64(
                src[0].numel() * 4)
            d["h"], d["w"], d["s"] = self.h, self.w, s
            self.prev_desc.append(torch.from_numpy(d.view(np.uint8).copy()).to(dev))
        self.parity = 0
        self.primed = False

    def tokenize(self, frames: torch.Tensor, g: int) -> None:
        tm = self.timer
        tm.begin("L_encode")
        self.model.encode_frames(frames[:g], self.s, codes=self.tok[:g], mask=self.mask[:g],
                                 idx=self.idx[:g])
        tm.end("L_encode")
        tm.begin("L_similarity")
        _lib.call("sst_similarity_gop", self.tok.data_ptr(), g, self.n, CHANNELS,
                  self.sim.data_ptr(), _dev.stream())
        tm.end("L_similarity")

    def decode(self, g: int, parity: int, arena: torch.Tensor | None = None,
               present: torch.Tensor | None = None) -> torch.Tensor:
        """K4 parse + reassemble, then the learned decoder; returns the
        [g, 9, h, w, 3] working-resolution frames."""
        st = _dev.stream()
        arena = self.arena if arena is None else arena
        npk = g * self.n_pkt_per_gop
        tm = self.timer
        tm.begin("K4_parse")
        _lib.call("sst_parse", arena.data_ptr(), self.offsets.data_ptr(),
                  self.lengths.data_ptr(), None if present is None else present.data_ptr(), npk,
                  self.info.data_ptr(), st)
        tm.end("K4_parse")
        # reassembly fused with the decoder's input stage: tokens go from the
        # winning packets straight to the bf16 input of the first conv
        tm.begin("K4_unpack_dec_in")
        _lib.call("sst_lt_unpack_dec_in", arena.data_ptr(), self.offsets.data_ptr(),
                  self.info.data_ptr(), self.target.data_ptr(), npk, g, self.Ht, self.Wt,
                  self.exp_gop.data_ptr(), self.winner.data_ptr(), self.stats.data_ptr(),
                  self.dec_ws.data_ptr(), self.dec_x.data_ptr(), st)
        tm.end("K4_unpack_dec_in")
        tm.begin("L_decode")
        self.model.decode_inputs(self.dec_x[:g], (self.h, self.w), frames=self.frames9[parity][:g])
        tm.end("L_decode")
        return self.frames9[parity][:g]

    def reconstruct(self, g: int, parity: int, out: torch.Tensor, blend: bool = True) -> None:
        """K5 for 9 distinct frames: upscale frames9[parity][:g] to
        [g, 9, H, W, 3] and, when ``blend``, mix frames 0..n-1 with the
        previous step's GoP in the same slot (frames9[1 - parity])."""
        check_gop_tensor(out, g, self.H, self.W, "out")
        self.timer.begin("K5_upscale_blend")
        prev = self.prev_desc[parity].data_ptr() if blend else None
        _lib.call("sst_upscale_blend9", self.frames9[parity].data_ptr(), g, self.h, self.w,
                  self.s, self.H, self.W, prev, self.blend_n, out.data_ptr(), _dev.stream())
        self.timer.end("K5_upscale_blend")

    def step(self, frames: torch.Tensor, out: torch.Tensor, g: int, drop_k: int = 0,
             present: torch.Tensor | None = None) -> None:
        """One GoP of each of g streams (slot j = stream j) through the learned
        codec: sender, then receiver; from the second step on, frames 0..n-1
        blend with the stream's previous GoP (codec.py:278-296)."""
        par = self.parity
        self.tokenize(frames, g)
        self.select_and_pack(g, drop_k)
        self.decode(g, par, present=present)
        self.reconstruct(g, par, out, blend=self.primed)
        self.parity ^= 1
        self.primed = True


class GraphedLearnedGopCodec:
    """CUDA-graph replay of one LearnedGopCodec step (learned encode + FSQ,
    similarity, drop, packetise, parse, packets -> decoder input, learned
    decode, K5-9) for a fixed batch, fixed device buffers and one geometry --
    the single-stream, one-GoP-in-flight regime, where ~30 launches per GoP
    are host-bound.  Three graphs, as in ``pipeline.GraphedGopCodec``: the
    first GoP (no blending) and the two steady-state parities (each blends
    with the decoded frames the other parity wrote)."""

    def __init__(self, codec: LearnedGopCodec, g: int, frames: torch.Tensor, out: torch.Tensor,
                 drop_k: int = 0):
        check_gop_tensor(frames, g, codec.H, codec.W, "frames")
        check_gop_tensor(out, g, codec.H, codec.W, "out")
        self.codec, self.g, self.frames, self.out, self.drop_k = codec, g, frames, out, drop_k
        codec.set_gop_ids([0] * g)
        plan = ((0, False), (1, True), (0, True))
        side = torch.cuda.Stream(device=frames.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):                # warm-up outside capture
            for par, blend in plan:
                self._body(par, blend)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graphs = []
        for par, blend in plan:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                self._body(par, blend)
            self.graphs.append(gr)
        self.k = 0

    def _body(self, parity: int, blend: bool) -> None:
        c = self.codec
        c.tokenize(self.frames, self.g)
        c.select_and_pack(self.g, self.drop_k)
        c.decode(self.g, parity)
        c.reconstruct(self.g, parity, self.out, blend=blend)

    def step(self, gop_ids) -> None:
        """Encode ... reconstruct the GoPs currently in ``frames`` into ``out``."""
        self.codec.set_gop_ids(gop_ids)
        idx = 0 if self.k == 0 else (1 if self.k % 2 == 1 else 2)
        self.graphs[idx].replay()
        self.k += 1
