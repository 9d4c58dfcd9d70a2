"""Batched, device-resident codec path: the B200 hot path behind the
reference API.

``GopCodec`` runs a batch of GoPs of one geometry (H, W, s) through

    K1 sst_encode        scale_gop(down) + encode_gop + token_similarity
    K2 sst_select_drop   build_drop_mask + apply_token_mask (P layer)
    K3 sst_packetize     packetize_tokens + TokenPacket.to_bytes (I rows, P rows)
    K4 sst_parse +       parse_packet + reassemble x2 + decode_gop
       sst_unpack_decode (mask-aware decoder reads tokens out of the packets)
    K5 sst_upscale_blend scale_gop(up, crop) + blend_boundary, 9 frames out

which is the reference's per-GoP composition (session.py:134-170 sender,
session.py:323-348 receiver) minus the emulated network.  All buffers are
allocated once; every call is stream-ordered on torch's current stream.

``StreamBank`` keeps many independent streams (each with its own previous
GoP for boundary blending and its own per-GoP scale) and routes every step's
GoPs to one ``GopCodec`` per scale.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib
from .transport import token_packet_wire_size

GOP = 9
CHANNELS = 12


def _cdiv(a: int, b: int) -> int:
    return -(-a // b)


def check_gop_tensor(t: torch.Tensor, g: int, H: int, W: int, what: str,
                     dtypes=(torch.float32,)) -> None:
    """The kernels address [g][9][H][W][3] float32 (or, where ``dtypes``
    allows it, raw-rgb24 uint8) by raw pointer: reject anything else (a
    non-contiguous view, e.g. a transposed numpy array wrapped by
    torch.from_numpy, would otherwise be read in the wrong order)."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor")
    if t.dtype not in dtypes:
        want = " or ".join(str(d).replace("torch.", "") for d in dtypes)
        raise ValueError(f"{what} must be {want}, got {t.dtype}")
    if t.dim() != 5 or tuple(t.shape[1:]) != (GOP, H, W, 3) or t.shape[0] < g:
        raise ValueError(f"{what} must be [>= {g}, {GOP}, {H}, {W}, 3], got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous (call .contiguous())")


class StageTimer:
    """CUDA-event timing of each kernel stage on the launching (current) stream."""

    def __init__(self, lead_cycles: int = 0):
        self.pairs: dict = {}
        self._open: dict = {}
        # lead_cycles > 0: enqueue a GPU spin of that many cycles before each
        # begin event so the host runs ahead and the event pair brackets the
        # kernel alone (no launch / host gap inside the measured interval)
        self.lead_cycles = lead_cycles

    def begin(self, name: str) -> None:
        if self.lead_cycles:
            torch.cuda._sleep(self.lead_cycles)
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self._open[name] = ev

    def end(self, name: str) -> None:
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.pairs.setdefault(name, []).append((self._open.pop(name), ev))

    def reset(self) -> None:
        self.pairs.clear()
        self._open.clear()

    def summary(self) -> dict:
        """{stage: (total_ms, launches)} -- call after synchronising."""
        return {k: (sum(a.elapsed_time(b) for a, b in v), len(v)) for k, v in self.pairs.items()}


class _NoTimer:
    def begin(self, name):
        pass

    def end(self, name):
        pass


_NO_TIMER = _NoTimer()


class GopCodec:
    """Device buffers + kernel launches for up to ``g_max`` GoPs of (H, W, s)."""

    def __init__(self, g_max: int, H: int, W: int, s: int, blend_n: int = 2):
        if s not in (2, 3):
            raise ValueError(f"scale must be 2 or 3, got {s}")
        dev = _dev.device()
        self.g_max, self.H, self.W, self.s, self.blend_n = g_max, H, W, s, blend_n
        self.h, self.w = _cdiv(H, s), _cdiv(W, s)
        self.Ht, self.Wt = _cdiv(self.h, 8), _cdiv(self.w, 8)
        if self.Ht > 0xFFFF:
            raise ValueError(f"matrix has {self.Ht} rows; the row index field is 16-bit")
        n = self.Ht * self.Wt
        self.slot = (token_packet_wire_size(self.Wt, CHANNELS) + 15) & ~15
        self.n_pkt_per_gop = 2 * self.Ht
        G = g_max
        f64, u8, i32 = torch.float64, torch.uint8, torch.int32
        self.tok = torch.empty((G, 2, self.Ht, self.Wt, CHANNELS), dtype=f64, device=dev)
        self.sim = torch.empty((G, self.Ht, self.Wt), dtype=f64, device=dev)
        # token masks: the I half stays all-true (encode_gop, codec.py:155-157);
        # the P half is assigned by K2 (P := not dropped), so no per-step reset
        self.mask = torch.ones((G, 2, self.Ht, self.Wt), dtype=u8, device=dev)
        self._p_mask_dirty = False
        self.drop = torch.zeros((G, self.Ht, self.Wt), dtype=u8, device=dev)
        self.k = torch.zeros((G,), dtype=i32, device=dev)
        self._k_val = 0
        self.kind = torch.tensor([0, 1] * G, dtype=u8, device=dev)
        # per-GoP ids, one buffer so a step's ids arrive with ONE host->device
        # copy (no fill kernels): [exp_gop (G) | gop_id per matrix (2G)], u32 bits
        self._ids = torch.zeros((3 * G,), dtype=torch.int32, device=dev)
        self.exp_gop = self._ids[:G]
        self.gop_id = self._ids[G:]
        self.scale = torch.full((2 * G,), s, dtype=u8, device=dev)
        npk = G * self.n_pkt_per_gop
        self.arena = torch.empty((npk, self.slot), dtype=u8, device=dev)
        self.lengths = torch.empty((npk,), dtype=i32, device=dev)
        self.offsets = torch.arange(npk, dtype=torch.int64, device=dev) * self.slot
        self.info = torch.empty((npk * _lib.INFO_BYTES,), dtype=u8, device=dev)
        # arrival order = slot order: packet p of GoP g targets matrix 2g + kind
        tgt = np.repeat(np.arange(G) * 2, self.n_pkt_per_gop) + \
            np.tile(np.repeat([0, 1], self.Ht), G)
        self.target = torch.from_numpy(tgt.astype(np.int32)).to(dev)
        self.winner = torch.empty((2 * G * self.Ht,), dtype=torch.int32, device=dev)
        self.stats = torch.empty((2 * G * 2,), dtype=i32, device=dev)
        ws = _lib.load().sst_unpack_decode_workspace(G, self.Ht, self.Wt)
        self.dec_ws = torch.empty((ws,), dtype=u8, device=dev)
        # double-buffered working images so the next step can still read the
        # previous GoP's P image for boundary blending
        self.img = [torch.empty((G, 2, self.h, self.w, 3), dtype=torch.float32, device=dev)
                    for _ in range(2)]
        # decoder-fused reconstruction (sst_unpack_tokens + sst_upscale_blend_tok):
        # double-buffered dequantised token matrices + P validity, allocated on
        # first use
        self.tokq = None
        self.pvalid = None
        self.n = n
        self.timer = _NO_TIMER
        self._id_ring = _DescRing(3 * G * 4)

    # -- helpers -------------------------------------------------------
    def drop_k(self, rate: float) -> int:
        return int(np.floor(rate * self.n + 0.5))

    def set_gop_ids(self, gop_ids) -> None:
        """Per-GoP gop_id of the next batch: one asynchronous host->device copy
        from a pinned staging ring into the id buffer (no kernel launch; a
        pageable copy would synchronise the stream)."""
        ids = np.asarray(gop_ids, dtype=np.uint32)
        g = ids.size
        G = self.g_max
        raw = np.zeros(3 * G, dtype=np.uint32)
        raw[:g] = ids
        raw[G:G + 2 * g] = np.repeat(ids, 2)
        self._id_ring.copy_to(raw.view(np.uint8), self._ids)

    # -- sender --------------------------------------------------------
    def encode(self, frames: torch.Tensor, g: int, drop_k: int = 0,
               work: torch.Tensor | None = None) -> None:
        """K1 + K2 + K3 for frames[:g] ([g, 9, H, W, 3] float32 -- or uint8
        raw-rgb24, sample q meaning float32(q) / 255 as load_raw_video reads
        it (video.py:130-135) -- contiguous); `work` ([>= g, 9, h, w, 3]
        float32) also receives the working frames."""
        self.tokenize(frames, g, work)
        self.select_and_pack(g, drop_k)

    def tokenize(self, frames: torch.Tensor, g: int, work: torch.Tensor | None = None) -> None:
        """K1: downscale + tokenize + similarity (+ the working frames when
        `work` is given: the residual layer's input, no second frame read)."""
        tm = self.timer
        check_gop_tensor(frames, g, self.H, self.W, "frames", (torch.float32, torch.uint8))
        if work is not None:
            check_gop_tensor(work, g, self.h, self.w, "work")
        tm.begin("K1_encode")
        _lib.call("sst_encode_u8" if frames.dtype == torch.uint8 else "sst_encode_work",
                  frames.data_ptr(), g, self.H, self.W, self.s,
                  self.tok.data_ptr(), self.sim.data_ptr(),
                  None if work is None else work.data_ptr(), _dev.stream())
        tm.end("K1_encode")

    def select_and_pack(self, g: int, drop_k: int = 0) -> None:
        """K2 (intelligent drop) + K3 (quantise, packetise, CRC)."""
        st = _dev.stream()
        tm = self.timer
        if drop_k > 0 or self._p_mask_dirty:
            if drop_k != self._k_val:
                self.k.fill_(drop_k)           # only when the drop count changes
                self._k_val = drop_k
            # K2 assigns the P mask (P := not dropped): k = 0 just restores it
            tm.begin("K2_select_drop")
            _lib.call("sst_select_drop", self.sim.data_ptr(), self.tok.data_ptr(),
                      self.mask.data_ptr(), g, self.Ht, self.Wt, self.k.data_ptr(),
                      self.drop.data_ptr(), st)
            tm.end("K2_select_drop")
            self._p_mask_dirty = drop_k > 0
        tm.begin("K3_packetize")
        _lib.call("sst_packetize", self.tok.data_ptr(), self.mask.data_ptr(), 2 * g, self.Ht,
                  self.Wt, CHANNELS, self.kind.data_ptr(), self.gop_id.data_ptr(),
                  self.scale.data_ptr(), self.arena.data_ptr(), self.slot,
                  self.lengths.data_ptr(), st)
        tm.end("K3_packetize")

    # -- receiver ------------------------------------------------------
    def decode(self, g: int, parity: int, arena: torch.Tensor | None = None,
               present: torch.Tensor | None = None, fused: bool = False) -> torch.Tensor | None:
        """K4: parse + first-wins reassembly + mask-aware decode of the packet
        slots of g GoPs; returns the [g, 2, h, w, 3] working images.  fused:
        stop before the IDCT -- the dequantised token matrices and P validity
        go to ``tokq[parity]`` / ``pvalid[parity]`` for ``reconstruct(...,
        fused=True)``, which decodes inside K5 (returns None)."""
        st = _dev.stream()
        arena = self.arena if arena is None else arena
        npk = g * self.n_pkt_per_gop
        img = self.img[parity]
        tm = self.timer
        tm.begin("K4_parse")
        _lib.call("sst_parse", arena.data_ptr(), self.offsets.data_ptr(),
                  self.lengths.data_ptr(), None if present is None else present.data_ptr(), npk,
                  self.info.data_ptr(), st)
        tm.end("K4_parse")
        if fused:
            if self.tokq is None:
                dev = _dev.device()
                self.tokq = [torch.empty((self.g_max, 2, self.Ht, self.Wt, CHANNELS),
                                         dtype=torch.float64, device=dev) for _ in range(2)]
                self.pvalid = [torch.empty((self.g_max, self.Ht, self.Wt), dtype=torch.uint8,
                                           device=dev) for _ in range(2)]
            tm.begin("K4_unpack_decode")
            _lib.call("sst_unpack_tokens", arena.data_ptr(), self.offsets.data_ptr(),
                      self.info.data_ptr(), self.target.data_ptr(), npk, g, self.Ht, self.Wt,
                      self.exp_gop.data_ptr(), self.winner.data_ptr(), self.stats.data_ptr(),
                      self.dec_ws.data_ptr(), self.tokq[parity].data_ptr(),
                      self.pvalid[parity].data_ptr(), st)
            tm.end("K4_unpack_decode")
            return None
        tm.begin("K4_unpack_decode")
        _lib.call("sst_unpack_decode", arena.data_ptr(), self.offsets.data_ptr(),
                  self.info.data_ptr(), self.target.data_ptr(), npk, g, self.Ht, self.Wt, self.h,
                  self.w, self.exp_gop.data_ptr(), self.winner.data_ptr(), self.stats.data_ptr(),
                  self.dec_ws.data_ptr(), img.data_ptr(), st)
        tm.end("K4_unpack_decode")
        return img[:g]

    # -- reconstruction ------------------------------------------------
    def reconstruct(self, g: int, parity: int, out: torch.Tensor,
                    prev: torch.Tensor | None = None, fused: bool = False) -> None:
        """K5: [g, 9, H, W, 3] float32 output frames -- or uint8 raw-rgb24,
        each sample quantised as write_raw_video does (video.py:139-143);
        prev = device SstPrevDesc[g] as uint8 bytes (or None: no blending)."""
        check_gop_tensor(out, g, self.H, self.W, "out", (torch.float32, torch.uint8))
        if fused:
            # K5 with decode_gop fused: prev = device SstPrevTokDesc[g] bytes
            if out.dtype != torch.float32:
                raise ValueError("the decoder-fused reconstruction writes float32 frames")
            self.timer.begin("K5_upscale_blend")
            _lib.call("sst_upscale_blend_tok", self.tokq[parity].data_ptr(),
                      self.pvalid[parity].data_ptr(), g, self.Ht, self.Wt, self.h, self.w, self.s,
                      self.H, self.W, None if prev is None else prev.data_ptr(), self.blend_n,
                      out.data_ptr(), _dev.stream())
            self.timer.end("K5_upscale_blend")
            return
        self.timer.begin("K5_upscale_blend")
        _lib.call("sst_upscale_blend_u8" if out.dtype == torch.uint8 else "sst_upscale_blend",
                  self.img[parity].data_ptr(), g, self.h, self.w, self.s,
                  self.H, self.W, None if prev is None else prev.data_ptr(), self.blend_n,
                  out.data_ptr(), _dev.stream())
        self.timer.end("K5_upscale_blend")

    def packet_status(self, g: int) -> np.ndarray:
        info = _dev.d2h(self.info[: g * self.n_pkt_per_gop * _lib.INFO_BYTES])
        return info.view(_lib.INFO_DTYPE)["status"]


class _DescRing:
    """Pinned-host -> device staging for small per-step descriptor tables.
    A slot is reused only after the kernel that consumed it has completed
    (CUDA event), so the host may run several steps ahead of the GPU."""

    def __init__(self, nbytes: int, slots: int = 4):
        dev = _dev.device()
        self.host = [torch.empty((nbytes,), dtype=torch.uint8, pin_memory=True) for _ in range(slots)]
        self.dev = [torch.empty((nbytes,), dtype=torch.uint8, device=dev) for _ in range(slots)]
        self.events = [None] * slots
        self.i = 0

    def stage(self, raw: np.ndarray) -> tuple:
        j = self.i
        self.i = (self.i + 1) % len(self.host)
        if self.events[j] is not None:
            self.events[j].synchronize()
        n = raw.nbytes
        self.host[j][:n].copy_(torch.from_numpy(raw.view(np.uint8)))
        self.dev[j][:n].copy_(self.host[j][:n], non_blocking=True)
        return self.dev[j], j

    def release(self, j: int) -> None:
        ev = torch.cuda.Event()
        ev.record()
        self.events[j] = ev

    def copy_to(self, raw: np.ndarray, dst: torch.Tensor) -> None:
        """Stage ``raw`` in the next pinned slot and copy it straight into the
        device tensor ``dst`` (stream-ordered, no kernel)."""
        j = self.i
        self.i = (self.i + 1) % len(self.host)
        if self.events[j] is not None:
            self.events[j].synchronize()
        n = raw.nbytes
        self.host[j][:n].copy_(torch.from_numpy(raw.view(np.uint8)))
        dst.view(torch.uint8)[:n].copy_(self.host[j][:n], non_blocking=True)
        self.release(j)


class StreamBank:
    """``n_streams`` independent streams of (H, W) video; each step encodes,
    transports and reconstructs one GoP per stream.  Streams may change scale
    from GoP to GoP (variable-resolution mode); boundary blending always uses
    the stream's previous reconstruction, at whatever scale it was coded."""

    def __init__(self, n_streams: int, H: int, W: int, scales=(2, 3), blend_n: int = 2,
                 concurrent_groups: bool = True, priority_middle: bool = True,
                 fused: bool = False):
        if not 1 <= blend_n <= 8:                 # CodecConfig, codec.py:41-42
            raise ValueError(f"blend width must be in [1, 8], got {blend_n}")
        # fused: decode_gop runs inside the reconstruction (K4 stops at the
        # dequantised tokens, K5 decodes its windows in smem); float32 output
        # frames only, rows of an even number of floats (8-byte stores)
        self.fused = bool(fused) and (W * 3) % 2 == 0
        self.n, self.H, self.W, self.blend_n = n_streams, H, W, blend_n
        self.codecs = {s: GopCodec(n_streams, H, W, s, blend_n) for s in scales}
        # blend_n <= 4: K5 recomputes the previous GoP's (unblended) tail from
        # its working image.  blend_n >= 5 reaches back into frames the
        # previous blend already changed (frame 9-n+i-1 < n), so each stream
        # keeps its last full-resolution output instead and blends after K5,
        # sequentially per stream (codec.py:278-296).
        self.prev_out = None
        self.has_prev = [False] * n_streams
        self.prev_host = np.zeros(n_streams, dtype=_lib.PREV_DTYPE)
        self.rings = {s: _DescRing(n_streams * max(_lib.PREV_BYTES, _lib.PREVTOK_BYTES))
                      for s in scales}
        self.prev_tok_host = np.zeros(n_streams, dtype=_lib.PREVTOK_DTYPE)
        # each scale group runs on its own CUDA stream so the latency-bound
        # middle kernels of one group overlap the HBM-bound K1/K5 of the other
        self.group_streams = ({s: torch.cuda.Stream(device=_dev.device()) for s in scales}
                              if concurrent_groups else None)
        # the latency-bound middle kernels (drop, packetise, parse, decode) run
        # on a high-priority stream so their few CTAs are scheduled ahead of
        # other lanes' HBM-streaming K1/K5 CTAs instead of queueing behind them
        self.mid_stream = (torch.cuda.Stream(device=_dev.device(), priority=-10)
                           if priority_middle else None)
        self.step_idx = 0
        self.launches = 0          # kernels of this library launched by step()
        # where each stream's last P image lives: (scale, parity, slot) or None
        self.last = [None] * n_streams
        self._pending = None       # (frames, ids, gop_ids, drop_rate) between send / receive

    def step(self, frames_by_scale: dict, out_by_scale: dict, stream_ids_by_scale: dict,
             gop_ids_by_scale: dict, drop_rate: float = 0.0, present_by_scale: dict | None = None
             ) -> None:
        """One GoP for every stream.  ``frames_by_scale[s]`` holds the GoPs of
        the streams coded at scale s this step ([g, 9, H, W, 3]); outputs go to
        ``out_by_scale[s]`` in the same order.  ``present_by_scale[s]`` (uint8
        per packet slot, I rows then P rows per GoP) simulates network loss."""
        self._run(frames_by_scale, out_by_scale, stream_ids_by_scale, gop_ids_by_scale,
                  drop_rate, present_by_scale, send=True, receive=True)

    def send(self, frames_by_scale: dict, stream_ids_by_scale: dict, gop_ids_by_scale: dict,
             drop_rate: float = 0.0) -> None:
        """Sender half of ``step``: encode, drop and packetise one GoP per
        stream into the packet arena.  ``receive`` must follow before the
        next ``send`` (it consumes the arena); in between, other work may run
        on the stream -- e.g. a pipelined caller receives GoP k, then sends
        GoP k + 1, so its HBM-bound encode / reconstruction kernels sit on
        either side of the latency-bound middle ones."""
        self._run(frames_by_scale, None, stream_ids_by_scale, gop_ids_by_scale, drop_rate,
                  None, send=True, receive=False)

    def receive(self, out_by_scale: dict, present_by_scale: dict | None = None) -> None:
        """Receiver half of ``step`` for the GoPs of the last ``send``."""
        if self._pending is None:
            raise RuntimeError("receive() without a pending send()")
        frames_by_scale, ids, gop_ids, drop_rate = self._pending
        self._run(frames_by_scale, out_by_scale, ids, gop_ids, drop_rate, present_by_scale,
                  send=False, receive=True)

    def _run(self, frames_by_scale, out_by_scale, stream_ids_by_scale, gop_ids_by_scale,
             drop_rate, present_by_scale, send: bool, receive: bool) -> None:
        parity = self.step_idx & 1
        main = torch.cuda.current_stream()
        joined = []
        for s, frames in frames_by_scale.items():
            codec = self.codecs[s]
            ids = stream_ids_by_scale[s]
            g = len(ids)
            if g == 0:
                continue
            gs = self.group_streams[s] if self.group_streams and len(frames_by_scale) > 1 else main
            if gs is not main:
                gs.wait_stream(main)
                joined.append(gs)
            with torch.cuda.stream(gs):
                mid = self.mid_stream if self.mid_stream is not None else gs
                if send:
                    codec.set_gop_ids(gop_ids_by_scale[s])
                    codec.tokenize(frames, g)
                    if mid is not gs:
                        mid.wait_stream(gs)
                    with torch.cuda.stream(mid):
                        codec.select_and_pack(g, codec.drop_k(drop_rate))
                    # K1 + K2 (if dropping) + K3
                    self.launches += 1 + (1 if codec.drop_k(drop_rate) > 0 else 0) + 1
                if receive:
                    present = None if present_by_scale is None else present_by_scale.get(s)
                    if mid is not gs:
                        mid.wait_stream(gs)
                    if self.fused and out_by_scale[s].dtype != torch.float32:
                        raise ValueError("a fused StreamBank writes float32 frames "
                                         "(StreamBank(fused=False) for raw-rgb24 output)")
                    with torch.cuda.stream(mid):
                        codec.decode(g, parity, present=present, fused=self.fused)
                    if mid is not gs:
                        gs.wait_stream(mid)
                    # K4 parse + 5 (init/route/dups/rowprep/decode) + K5
                    self.launches += 1 + 5 + 1
                    if self.blend_n <= 4:
                        staged = self._prev_descs(s, ids)
                        codec.reconstruct(g, parity, out_by_scale[s],
                                          None if staged is None else staged[0],
                                          fused=self.fused)
                        if staged is not None:
                            self.rings[s].release(staged[1])
                    else:
                        if out_by_scale[s].dtype != torch.float32:
                            # the n >= 5 blend reads the previous float32 output back
                            raise ValueError("blend widths 5..8 need float32 output frames")
                        codec.reconstruct(g, parity, out_by_scale[s], None, fused=self.fused)
                        self._blend_wide(ids, out_by_scale[s])
                elif mid is not gs:
                    gs.wait_stream(mid)
        for gs in joined:
            main.wait_stream(gs)
        if not receive:
            self._pending = (frames_by_scale, stream_ids_by_scale, gop_ids_by_scale, drop_rate)
            return
        self._pending = None
        for s, ids in stream_ids_by_scale.items():
            for slot, sid in enumerate(ids):
                self.last[sid] = (s, parity, slot)
        self.step_idx += 1

    def _blend_wide(self, ids, out: torch.Tensor) -> None:
        """blend_boundary for n >= 5 against each stream's previous output,
        then keep this output as the next GoP's previous (stream-ordered)."""
        if self.prev_out is None:
            self.prev_out = torch.empty((self.n, GOP, self.H, self.W, 3), dtype=torch.float32,
                                        device=_dev.device())
        st = _dev.stream()
        for j, sid in enumerate(ids):
            if self.has_prev[sid]:
                _lib.call("sst_blend", self.prev_out[sid].data_ptr(), out[j].data_ptr(), 1,
                          self.H, self.W, self.blend_n, out[j].data_ptr(), st)
                self.launches += 1
            self.prev_out[sid].copy_(out[j])
            self.has_prev[sid] = True

    def set_timer(self, timer) -> None:
        for c in self.codecs.values():
            c.timer = timer if timer is not None else _NO_TIMER

    def _prev_descs(self, s: int, ids):
        if all(self.last[i] is None for i in ids):
            return None
        if self.fused:
            # the previous GoP's token matrices + P validity (SstPrevTokDesc)
            rec = self.prev_tok_host[:len(ids)]
            rec[:] = 0
            for j, sid in enumerate(ids):
                loc = self.last[sid]
                if loc is None:
                    continue
                ps, par, slot = loc
                c = self.codecs[ps]
                rec[j]["tok"] = c.tokq[par][slot].data_ptr()
                rec[j]["pvalid"] = c.pvalid[par][slot].data_ptr()
                rec[j]["h"], rec[j]["w"], rec[j]["s"] = c.h, c.w, ps
                rec[j]["Ht"], rec[j]["Wt"] = c.Ht, c.Wt
            return self.rings[s].stage(rec)
        rec = self.prev_host[:len(ids)]
        rec[:] = 0
        for j, sid in enumerate(ids):
            loc = self.last[sid]
            if loc is None:
                continue
            ps, par, slot = loc             # the previous GoP's scale, not this one's
            c = self.codecs[ps]
            img = c.img[par]
            rec[j]["p_img"] = img.data_ptr() + ((slot * 2 + 1) * c.h * c.w * 3) * 4
            rec[j]["h"], rec[j]["w"], rec[j]["s"] = c.h, c.w, ps
        return self.rings[s].stage(rec)


class GraphedGopCodec:
    """CUDA-graph replay of one GopCodec step (encode, drop, packetise, parse,
    decode, reconstruct + blend) for a fixed batch, fixed device buffers and
    one geometry -- the launch-bound regime (a single stream, one GoP in
    flight).  Three graphs are captured: the first GoP (no blending) and the
    two parities of the steady state (each blends with the working images
    the other parity wrote).  Per step the host only refreshes the GoP ids
    (device fills) and replays one graph."""

    def __init__(self, codec: GopCodec, g: int, frames: torch.Tensor, out: torch.Tensor,
                 drop_k: int = 0):
        check_gop_tensor(frames, g, codec.H, codec.W, "frames")
        check_gop_tensor(out, g, codec.H, codec.W, "out")
        self.codec, self.g, self.frames, self.out, self.drop_k = codec, g, frames, out, drop_k
        dev = frames.device
        self.prev = []
        for par in range(2):
            d = np.zeros(g, dtype=_lib.PREV_DTYPE)
            img = codec.img[1 - par]
            for j in range(g):
                d[j]["p_img"] = img.data_ptr() + ((j * 2 + 1) * codec.h * codec.w * 3) * 4
                d[j]["h"], d[j]["w"], d[j]["s"] = codec.h, codec.w, codec.s
            self.prev.append(torch.from_numpy(d.view(np.uint8).copy()).to(dev))
        codec.set_gop_ids([0] * g)
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):                # warm-up outside capture
            for par, prev in ((0, None), (1, self.prev[1]), (0, self.prev[0])):
                self._body(par, prev)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graphs = []
        for par, prev in ((0, None), (1, self.prev[1]), (0, self.prev[0])):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                self._body(par, prev)
            self.graphs.append(gr)
        self.k = 0

    def _body(self, parity: int, prev) -> None:
        c = self.codec
        c.tokenize(self.frames, self.g)
        c.select_and_pack(self.g, self.drop_k)
        c.decode(self.g, parity)
        c.reconstruct(self.g, parity, self.out, prev)

    def step(self, gop_ids) -> None:
        self.codec.set_gop_ids(gop_ids)
        idx = 0 if self.k == 0 else (1 if self.k % 2 == 1 else 2)
        self.graphs[idx].replay()
        self.k += 1


class GraphedStreamBank:
    """One stream, variable resolution (per-GoP scale), one GoP in flight,
    every step replayed as a CUDA graph -- the latency case (real-time single
    stream), where the ~14 launches of an eager step cost more than their
    kernels.  Same semantics as ``StreamBank(1, H, W)``: GoP k is coded at
    its own scale and blended with the stream's previous reconstruction,
    whatever scale that had.  One graph per (scale, step parity, previous
    scale or none): encode + drop + packetise + parse + decode + K5 with the
    previous GoP's P image (the other parity's working image of the codec of
    its scale) as the blend source.  Input frames are read from ``frames``
    and reconstructions written to ``out`` (fixed device buffers)."""

    def __init__(self, H: int, W: int, frames: torch.Tensor, out: torch.Tensor,
                 drop_rate: float = 0.0, scales=(2, 3), blend_n: int = 2):
        if blend_n > 4:
            raise ValueError("the graphed bank blends at most 4 frames (K5 fused blend)")
        check_gop_tensor(frames, 1, H, W, "frames")
        check_gop_tensor(out, 1, H, W, "out")
        self.frames, self.out, self.scales = frames, out, tuple(scales)
        self.codecs = {s: GopCodec(1, H, W, s, blend_n) for s in scales}
        self.drop_k = {s: c.drop_k(drop_rate) for s, c in self.codecs.items()}
        dev = frames.device
        # prev[(ps, par)]: the previous GoP coded at scale ps, whose working
        # images are codecs[ps].img[par]
        self.prev = {}
        for ps, c in self.codecs.items():
            for par in range(2):
                d = np.zeros(1, dtype=_lib.PREV_DTYPE)
                d[0]["p_img"] = c.img[par].data_ptr() + c.h * c.w * 3 * 4
                d[0]["h"], d[0]["w"], d[0]["s"] = c.h, c.w, ps
                self.prev[(ps, par)] = torch.from_numpy(d.view(np.uint8).copy()).to(dev)
        plan = [(s, par, ps) for s in scales for par in range(2) for ps in (None,) + tuple(scales)]
        for c in self.codecs.values():
            c.set_gop_ids([0])
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):                 # warm-up outside capture
            for key in plan:
                self._body(*key)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graphs = {}
        for key in plan:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                self._body(*key)
            self.graphs[key] = gr
        self.step_idx = 0
        self.last_scale = None

    def _body(self, s: int, parity: int, prev_scale) -> None:
        c = self.codecs[s]
        c.tokenize(self.frames, 1)
        c.select_and_pack(1, self.drop_k[s])
        c.decode(1, parity)
        prev = None if prev_scale is None else self.prev[(prev_scale, 1 - parity)]
        c.reconstruct(1, parity, self.out, prev)

    def step(self, s: int, gop_id: int) -> None:
        """Code the GoP now in ``frames`` at scale s into ``out``."""
        par = self.step_idx & 1
        self.codecs[s].set_gop_ids([gop_id])
        self.graphs[(s, par, self.last_scale)].replay()
        self.last_scale = s
        self.step_idx += 1
