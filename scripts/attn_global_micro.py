"""Int8 attention core alone, 32 x 1080p GoPs (s=3: 45 x 80 tokens per latent
frame, D = 256): windowed (sst_lt8_attn) vs global (sst_lt8_attn_global)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2602_03529_b200 import _dev, _lib
from paper_2602_03529_b200.learned_i8 import exp_table
G, Ht, Wt, D = 32, 45, 80, 256
dev = _dev.device()
qkv = torch.randint(-60, 60, (G, 2, Ht, Wt, 3 * D), dtype=torch.int8, device=dev)
out = torch.empty((G, 2, Ht, Wt, D), dtype=torch.int8, device=dev)
lut = torch.from_numpy(exp_table().copy()).to(dev)
for fn in ("sst_lt8_attn", "sst_lt8_attn_global"):
    def run():
        _lib.call(fn, qkv.data_ptr(), G, Ht, Wt, D, 9, lut.data_ptr(), out.data_ptr(), _dev.stream())
    for _ in range(2): run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5): run()
    e1.record(); torch.cuda.synchronize()
    print(f"{fn}: {e0.elapsed_time(e1) / 5:.3f} ms per launch")
