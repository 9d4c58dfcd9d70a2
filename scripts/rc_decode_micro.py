"""Range-decoder A/B and concurrency sweep: the bench's residual
workload (64 x 1080p GoPs at s=3, moving-square / noisy-motion streams) is
encoded once; its 64 payloads are then decoded by each decoder variant
(SST_RC: c = round-2 one-warp-in-256 cumulative-table kernel k_rc_decode_c,
x = the default k_rc_decode_x: one-warp CTAs, split cumulative table) with the
batch replicated x1 .. x8 (64 .. 512 streams in flight).  Measured (B200):
64 .. 512 streams take the same time (the coder is a per-stream latency
chain; 4-way concurrency per SM costs nothing), c 17.8 ms, x 15.5 ms.
Every decode is checked against the encoded scans.
Usage: python scripts/rc_decode_micro.py"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import bench
from paper_2602_03529_b200 import _dev, _lib
from paper_2602_03529_b200.pipeline import GopCodec

G, H, W, s = 64, 1080, 1920, 3
dev = _dev.device()
frames = bench.make_inputs(list(range(G)), H, W, dev, n_sets=1)[0]
c = GopCodec(G, H, W, s)
c.set_gop_ids([0] * G)
h, w = c.h, c.w
n = h * w * 3
st = _dev.stream()
work = torch.empty((G, 9, h, w, 3), device=dev)
avg = torch.empty((G, n), dtype=torch.float64, device=dev)
dense = torch.empty((G, n), dtype=torch.int16, device=dev)
mags = torch.empty((G, n), dtype=torch.float64, device=dev)
count = torch.empty((G,), dtype=torch.int32, device=dev)
cap = n // 2 + 64
idx_ws = torch.empty((G * n,), dtype=torch.int64, device=dev)
pay = torch.empty((G * cap,), dtype=torch.uint8, device=dev)
plen = torch.empty((G,), dtype=torch.int64, device=dev)
c.encode(frames, G, 0)
c.decode(G, 0)
_lib.call("sst_downscale", frames.data_ptr(), G * 9, H, W, s, work.data_ptr(), st)
_lib.call("sst_residual", work.data_ptr(), c.img[0].data_ptr(), G, h, w, 0.02, 1.0 / 127.0,
          avg.data_ptr(), dense.data_ptr(), mags.data_ptr(), count.data_ptr(), st)
_lib.call("sst_rc_encode", dense.data_ptr(), G, n, idx_ws.data_ptr(), pay.data_ptr(), cap,
          plen.data_ptr(), st)
torch.cuda.synchronize()
del frames, work, avg, mags, idx_ws
torch.cuda.empty_cache()
print(f"{G} GoPs: entries/GoP mean {count.float().mean().item():.0f} max {count.max().item()}, "
      f"payload bytes mean {plen.float().mean().item():.0f} max {plen.max().item()}")

offs0 = torch.arange(G, dtype=torch.int64, device=dev) * cap
res = {}
for mode in ("c", "x"):
    os.environ["SST_RC"] = mode
    for rep in (1, 2, 4, 8):
        Gr = G * rep
        offs = offs0.repeat(rep)
        lens = plen.repeat(rep)
        dec = torch.empty((Gr, n), dtype=torch.int16, device=dev)
        status = torch.empty((Gr,), dtype=torch.int32, device=dev)

        def run():
            _lib.call("sst_rc_decode", pay.data_ptr(), offs.data_ptr(), lens.data_ptr(), Gr, n,
                      dec.data_ptr(), status.data_ptr(), st)
        run()
        torch.cuda.synchronize()
        ok = bool((status == 0).all()) and bool(torch.equal(dec, dense.repeat(rep, 1)))
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            run()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        res[(mode, Gr)] = ms
        print(f"SST_RC={mode} streams {Gr:4d}: {ms:8.3f} ms  ({Gr / ms:7.2f} GoPs/ms)  exact={ok}",
              flush=True)
        del dec, status
os.environ.pop("SST_RC")
