"""Diagnostic: per-layer GPU vs oracle agreement for the learned tokenizer."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import learned_oracle as LO
from oracle.synth import make_clip
from paper_2602_03529_b200 import _dev
from paper_2602_03529_b200.learned import LearnedConfig, LearnedTokenizer, make_weights

cfg = LearnedConfig(dim=128, blocks=2, seed=0)
w = make_weights(cfg)
m = LearnedTokenizer(cfg, w)
clip = make_clip("moving-square", 640, 360, 9, seed=3)
fr = np.stack([clip.gop(0)])
dev = _dev.device()

# hook: capture intermediate GPU activations by re-running layers manually
import paper_2602_03529_b200.learned as L
acts = []
orig = m._conv
def spy(name, x, *a, **k):
    orig(name, x, *a, **k)
    torch.cuda.synchronize()
    o = k.get("out")
    if o is not None:
        acts.append((name, o.float().cpu().clone()))
m._conv = spy
codes, idx, mask, hw = m.encode_frames(torch.from_numpy(fr).to(dev), 1)

pI, pP, _ = LO.patchify(fr, 1)
h0 = LO.bf(LO.linear(pI, w["W"]["pe_i"], w["b"]["pe_i"]))
h1 = LO.bf(LO.linear(pP, w["W"]["pe_p"], w["b"]["pe_p"]))
h = torch.stack([h0, h1], 1)
def cmp(tag, g, o):
    d = (g - o).abs()
    rel = d / o.abs().clamp_min(1e-3)
    print(f"{tag:10s} exact {(g == o).float().mean().item():.5f} max_abs {d.max().item():.3e} max_rel {rel.max().item():.3e} mean_abs {d.mean().item():.3e}")
cmp("pe(after both)", acts[1][1], h)
# stage isolated: feed GPU's h into oracle for each block
hg = acts[1][1]
for i in range(cfg.blocks):
    u_o = LO.conv233(hg, w["W"][f"enc{i}_c1"], w["b"][f"enc{i}_c1"], act=True)
    u_g = acts[2 + 2 * i][1]
    cmp(f"enc{i}_c1", u_g, u_o)
    h_o = LO.conv233(u_g, w["W"][f"enc{i}_c2"], w["b"][f"enc{i}_c2"], residual=hg)
    h_g = acts[3 + 2 * i][1]
    cmp(f"enc{i}_c2", h_g, h_o)
    hg = h_g
# FSQ stage isolated
z = LO.linear(hg, w["W"]["head"], w["b"]["head"])[..., :12]
oc, oi = LO.fsq(z)
print("fsq stage-isolated idx agree", (idx.cpu().numpy() == oi.numpy()).all(-1).mean())
oc2, oi2, _, z2 = LO.encode(fr, 1, w, cfg.blocks)
print("e2e idx agree", (idx.cpu().numpy() == oi2).all(-1).mean(), "tokens", oi2.shape)
print("z e2e diff max", (z - z2).abs().max().item(), "z std", z2.std().item())
