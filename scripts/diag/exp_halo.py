import os, sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
from test_gpu_learned import _conv_gpu, _bf
from oracle import learned_oracle as LO
from paper_2602_03529_b200 import _lib
from paper_2602_03529_b200.learned import TAPS_233
rng = np.random.default_rng(1)
for shape, cin in [((2, 2, 16, 16, 64), 64), ((1, 2, 45, 80, 256), 256), ((2, 2, 13, 37, 64), 64)]:
    G, Tn, H, Wd, _ = shape
    x = _bf(rng.standard_normal(shape))
    W = _bf(rng.standard_normal((256, 18 * cin)) / np.sqrt(18 * cin)).numpy()
    b = _bf(rng.standard_normal(256) * 0.1).numpy()
    resid = _bf(rng.standard_normal((G, Tn, H, Wd, 256)))
    want = LO.conv233(x, W, b, act=True, residual=resid)
    for mode in ("p", "c"):
        os.environ["SST_LT_CONV"] = {"g": "generic", "h": "halo", "p": "persistent", "c": "cluster"}[mode]
        got = _conv_gpu(x, W, b, TAPS_233, 0, 2, _lib.LT_EPI_STORE, act=1, residual=resid)["out"]
        err = (got - want).abs()
        print(shape, "mode", mode, "exact", (got == want).float().mean().item(), "max err", err.max().item())
