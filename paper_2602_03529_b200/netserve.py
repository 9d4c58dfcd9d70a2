"""Batched sender / receiver around an emulated network.

``LinkedStreamBank`` serves many streams with one batched GPU codec
(``pipeline.StreamBank``: every stream's GoP encoded, dropped, packetised,
parsed, decoded and reconstructed in a handful of launches) while each
stream's row packets cross ITS OWN link -- any object with the reference
netem's interface (``transmit(nbytes, now) -> Delivered(delivery_time, ...)
| Dropped(reason)``, ``semstream.netem.EmulatedLink``, netem.py:145-199):
trace-paced delivery, seeded Bernoulli loss, propagation delay, bounded
queue.  Per GoP k the sender transmits the stream's packets at
``k * gop_period_ms`` in the reference's order (I rows, then P rows;
session.py:159-166) and the receiver decodes at
``k * gop_period_ms + playout_offset_ms`` (session.py:230-233) with exactly
the packets the link delivered by then: lost, queue-dropped and late rows
are absent (zero-filled, I-concealed; transport.py:274-305, codec.py:176-180).

Only packet SIZES leave the device (the link model needs nothing else); the
packet bytes stay in the device arena and the delivered set returns as a
per-packet ``present`` mask.  Not modelled: NACK-driven retransmission
(session.py:243-258) -- this is the open-loop serving path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev
from .pipeline import StreamBank


class LinkedStreamBank:
    """``n_streams`` streams of (H, W) video through a ``StreamBank``, one
    emulated link per stream (``links[stream_id]``)."""

    def __init__(self, n_streams: int, H: int, W: int, links, gop_period_ms: float = 300.0,
                 playout_offset_ms: float = 120.0, scales=(2, 3), blend_n: int = 2):
        if len(links) != n_streams:
            raise ValueError(f"need one link per stream ({n_streams}), got {len(links)}")
        self.bank = StreamBank(n_streams, H, W, scales=scales, blend_n=blend_n)
        self.links = list(links)
        self.period = float(gop_period_ms)
        self.offset = float(playout_offset_ms)
        self.stats = [dict(sent=0, delivered=0, lost=0, queue=0, late=0) for _ in links]

    def step(self, frames_by_scale: dict, out_by_scale: dict, stream_ids_by_scale: dict,
             gop_id: int, drop_rate: float = 0.0) -> dict:
        """One GoP (id ``gop_id``) of every stream.  Returns, per stream id,
        the per-packet delivery flags of this GoP (I rows then P rows)."""
        bank = self.bank
        gids = {s: [gop_id] * len(ids) for s, ids in stream_ids_by_scale.items()}
        bank.send(frames_by_scale, stream_ids_by_scale, gids, drop_rate)
        now = gop_id * self.period
        deadline = now + self.offset
        present_by_scale, delivered = {}, {}
        for s, ids in stream_ids_by_scale.items():
            g = len(ids)
            if g == 0:
                continue
            codec = bank.codecs[s]
            npk = codec.n_pkt_per_gop
            lengths = _dev.d2h(codec.lengths[:g * npk])          # the link needs sizes only
            keep = np.zeros(g * npk, dtype=np.uint8)
            for j, sid in enumerate(ids):
                link, st = self.links[sid], self.stats[sid]
                for p in range(npk):
                    st["sent"] += 1
                    out = link.transmit(int(lengths[j * npk + p]), now)
                    t = getattr(out, "delivery_time", None)
                    if t is None:
                        st["queue" if getattr(out, "reason", "") == "queue" else "lost"] += 1
                    elif t > deadline:
                        st["late"] += 1
                    else:
                        st["delivered"] += 1
                        keep[j * npk + p] = 1
                delivered[sid] = keep[j * npk:(j + 1) * npk].copy()
            present_by_scale[s] = torch.from_numpy(keep).to(codec.lengths.device)
        bank.receive(out_by_scale, present_by_scale)
        return delivered
