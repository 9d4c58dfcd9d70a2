import os, sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
from oracle import learned_oracle as LO
from paper_2602_03529_b200 import _dev, _lib
rng = np.random.default_rng(12)
for (G, H, W, D) in [(2, 8, 8, 128), (1, 8, 8, 256), (1, 13, 21, 128), (2, 13, 21, 256)]:
    qkv = LO.bf(torch.from_numpy(rng.standard_normal((G, 2, H, W, 3 * D)).astype(np.float32)))
    qd = qkv.to("cuda", torch.bfloat16).contiguous()
    want = LO.window_attention(qkv)
    for mode in ("simt", "tc"):
        os.environ["SST_LT_ATTN"] = mode
        out = torch.full((G, 2, H, W, D), 7.0, dtype=torch.bfloat16, device="cuda")
        _lib.call("sst_lt_attn", qd.data_ptr(), G, H, W, D, out.data_ptr(), _dev.stream())
        torch.cuda.synchronize()
        got = out.float().cpu()
        err = (got - want).abs()
        bad = err > 2 * 2 ** -7 * want.abs().clamp_min(1e-3)
        idx = bad.nonzero()
        print((G, H, W, D), mode, "bad", bad.float().mean().item(), "max", err.max().item(),
              "first bad", idx[:3].tolist(), "zero frac", (got == 0).float().mean().item())
