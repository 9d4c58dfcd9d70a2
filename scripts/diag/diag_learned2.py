"""(Experiment record: written against the reverted fp32-residual-stream variant,
which exposed an `out32` conv output.)  Where does end-to-end FSQ divergence come from?  Compare GPU vs oracle z
(pre-FSQ) and the stream after each encoder stage, e2e (no isolation)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import learned_oracle as LO
from oracle.synth import make_clip
from paper_2602_03529_b200 import _dev
from paper_2602_03529_b200.learned import LearnedConfig, LearnedTokenizer, make_weights
cfg = LearnedConfig(); w = make_weights(cfg); m = LearnedTokenizer(cfg, w)
fr = np.stack([make_clip("moving-square", 1920, 1080, 9, seed=1).gop(0)])
caps = []
orig = m._conv
def spy(name, x, *a, **k):
    orig(name, x, *a, **k); torch.cuda.synchronize()
    if k.get("out32") is not None: caps.append((name, k["out32"].clone().cpu()))
    elif k.get("out") is not None: caps.append((name, k["out"].float().clone().cpu()))
m._conv = spy
codes, idx, mask, hw = m.encode_frames(torch.from_numpy(fr).to(_dev.device()), 3)
Wm, bm = w["W"], w["b"]
pI, pP, _ = LO.patchify(fr, 3)
h = torch.stack([LO.linear(pI, Wm["pe_i"], bm["pe_i"]), LO.linear(pP, Wm["pe_p"], bm["pe_p"])], 1)
ref = {}
ref["pe_p"] = h.clone()
for i in range(cfg.blocks):
    u = LO.conv233(LO.bf(h), Wm[f"enc{i}_c1"], bm[f"enc{i}_c1"], act=True); ref[f"enc{i}_c1"] = u
    h = LO.conv233(u, Wm[f"enc{i}_c2"], bm[f"enc{i}_c2"], residual=h, round_bf16=False); ref[f"enc{i}_c2"] = h.clone()
qkv = LO.bf(LO.linear(LO.bf(h), Wm["enc_qkv"], bm["enc_qkv"])); ref["enc_qkv"] = qkv
o = LO.window_attention(qkv)
h = LO.linear(o, Wm["enc_proj"], bm["enc_proj"]) + h; ref["enc_proj"] = h.clone()
z = LO.linear(LO.bf(h), Wm["head"], bm["head"])[..., :12]
for name, g in caps:
    if name in ref:
        r = ref[name]; d = (g - r).abs()
        print(f"{name:10s} max {d.max().item():.3e} mean {d.mean().item():.3e} frac_diff {(d > 0).float().mean().item():.4f} scale {r.abs().mean().item():.3f}")
oc, oi = LO.fsq(z)
print("idx agree", (idx.cpu().numpy() == oi.numpy()).mean())
# z from the GPU's own final stream (isolate the head)
hg = caps[[n for n, _ in caps].index("enc_proj")][1]
zg = LO.linear(LO.bf(hg), Wm["head"], bm["head"])[..., :12]
print("z diff (oracle head on GPU stream vs oracle) max", (zg - z).abs().max().item(), "mean", (zg - z).abs().mean().item())
