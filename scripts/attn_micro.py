"""Fused qkv + window attention alone at the learned leg's shape (32 x 1080p
GoPs, s=3: 45 x 80 tokens x 2 latent frames, D=256): one-CTA-per-item vs the
persistent kernel, CUDA-event timed back-to-back launches."""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2602_03529_b200 import _dev, _lib
G, Ht, Wt, D = 32, 45, 80, 256
dev = _dev.device()
h = (torch.randn((G, 2, Ht, Wt, D), device=dev) * 0.5).to(torch.bfloat16)
w = (torch.randn((3 * D, D), device=dev) / 16).to(torch.bfloat16)
b = torch.randn(3 * D, device=dev) * 0.1
out = torch.empty_like(h)
tok = G * 2 * Ht * Wt
flops = 2 * tok * D * 3 * D + 2 * 2 * tok * 128 * 64 * (D // 64)   # qkv + S + PV (dense 128 keys)
for mode in ("fused", "persistent"):
    os.environ["SST_LT_ATTN"] = mode
    run = lambda: _lib.call("sst_lt_attn_fused", h.data_ptr(), w.data_ptr(), b.data_ptr(), G, Ht, Wt,
                            D, out.data_ptr(), _dev.stream())
    for _ in range(3): run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    n = 20
    e0.record()
    for _ in range(n): run()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{mode:10s} {ms:.3f} ms  {flops / ms / 1e9:.0f} TFLOP/s (qkv + dense-window S/PV)")
