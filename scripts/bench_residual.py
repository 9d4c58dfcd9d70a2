"""Residual layer + range coder on the GPU: G x 1080p GoPs at
s=3 through the proxy codec, then sender-side residual (downscale, residual vs
the decoded working images, sparsify, range-encode) and receiver-side
(range-decode, apply).  Usage: python scripts/bench_residual.py [G] [clip]"""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import bench
from paper_2602_03529_b200 import _dev, _lib
from paper_2602_03529_b200.pipeline import GopCodec
G = int(sys.argv[1]) if len(sys.argv) > 1 else 32
H, W, s = 1080, 1920, 3
dev = _dev.device()
frames = bench.make_inputs(list(range(G)), H, W, dev, n_sets=1)[0]
c = GopCodec(G, H, W, s)
c.set_gop_ids([0] * G)
h, w = c.h, c.w
n = h * w * 3
work = torch.empty((G, 9, h, w, 3), device=dev)
avg = torch.empty((G, n), dtype=torch.float64, device=dev)
dense = torch.empty((G, n), dtype=torch.int16, device=dev)
mags = torch.empty((G, n), dtype=torch.float64, device=dev)
count = torch.empty((G,), dtype=torch.int32, device=dev)
cap = n // 2 + 64
idx_ws = torch.empty((G * n,), dtype=torch.int64, device=dev)
pay = torch.empty((G * cap,), dtype=torch.uint8, device=dev)
plen = torch.empty((G,), dtype=torch.int64, device=dev)
dec = torch.empty((G, n), dtype=torch.int16, device=dev)
status = torch.empty((G,), dtype=torch.int32, device=dev)
offs = torch.arange(G, dtype=torch.int64, device=dev) * cap
st = _dev.stream()
def stage(name, fn, times):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); fn(); e1.record(); times.setdefault(name, []).append((e0, e1))
def step(times):
    stage("codec", lambda: (c.encode(frames, G, 0), c.decode(G, 0)), times)
    stage("downscale", lambda: _lib.call("sst_downscale", frames.data_ptr(), G * 9, H, W, s, work.data_ptr(), st), times)
    stage("residual", lambda: _lib.call("sst_residual", work.data_ptr(), c.img[0].data_ptr(), G, h, w, 0.02, 1.0 / 127.0,
                                        avg.data_ptr(), dense.data_ptr(), mags.data_ptr(), count.data_ptr(), st), times)
    stage("rc_encode", lambda: _lib.call("sst_rc_encode", dense.data_ptr(), G, n, idx_ws.data_ptr(), pay.data_ptr(), cap,
                                         plen.data_ptr(), st), times)
    stage("rc_decode", lambda: _lib.call("sst_rc_decode", pay.data_ptr(), offs.data_ptr(), plen.data_ptr(), G, n,
                                         dec.data_ptr(), status.data_ptr(), st), times)
    stage("apply", lambda: _lib.call("sst_apply_residual", c.img[0].data_ptr(), dec.data_ptr(), count.data_ptr(), G, h, w,
                                     1.0 / 127.0, st), times)
for _ in range(2): step({})
torch.cuda.synchronize()
times = {}
for _ in range(3): step(times)
torch.cuda.synchronize()
tot = 0
for k, v in times.items():
    ms = np.median([a.elapsed_time(b) for a, b in v]); tot += ms
    print(f"{k:10s} {ms:8.3f} ms")
print("entries per GoP", count.float().mean().item(), "payload bytes per GoP", plen.float().mean().item(),
      "decode ok", bool((status == 0).all().item()), "roundtrip", bool(torch.equal(dec, dense)))
print(f"total {tot:.3f} ms per {G} GoPs -> {G * 9 / tot * 1e3:.0f} frames/s")
