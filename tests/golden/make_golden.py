"""Generate tests/golden/golden.json from the LIVE reference implementation.

Run in the build container only (needs /root/reference):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Each case runs the reference's own per-GoP composition (
session.py:134-170 sender, session.py:323-348 receiver, netem replaced by a
seeded packet-loss set) and records SHA-256 digests of every intermediate
(bit-exact contract) plus small arrays.  The fixtures travel with the repo;
/root/reference does not.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "golden.json"

CASES = [
    # name, clip, W, H, frames, seed, scales (per GoP; 1 = direct encode), drop, loss
    dict(name="c1_ms256_s2", clip="moving-square", W=256, H=256, frames=17, seed=0,
         scales=[2, 2], drop=0.10, loss=0.0),
    dict(name="c1_ms256_direct", clip="moving-square", W=256, H=256, frames=17, seed=0,
         scales=[1, 1], drop=0.0, loss=0.0),
    dict(name="nm96x72_s3_drop30_loss30", clip="noisy-motion", W=96, H=72, frames=27, seed=3,
         scales=[3, 3, 3], drop=0.30, loss=0.30),
    dict(name="sg102x62_s3_drop25", clip="static-gradient", W=102, H=62, frames=9, seed=0,
         scales=[3], drop=0.25, loss=0.0),
    dict(name="sd250x170_s2_drop20_loss10", clip="static-detail", W=250, H=170, frames=18,
         seed=1, scales=[2, 2], drop=0.20, loss=0.10),
    dict(name="nf64x40_var", clip="noise-field", W=64, H=40, frames=36, seed=2,
         scales=[3, 2, 2, 3], drop=0.05, loss=0.05),
    dict(name="c2_ms720p_s3", clip="moving-square", W=1280, H=720, frames=33, seed=1,
         scales=[3, 3, 3, 3], drop=0.0, loss=0.0),
    dict(name="c3_ms1080p_var_drop10", clip="moving-square", W=1920, H=1080, frames=18, seed=0,
         scales=[3, 2], drop=0.10, loss=0.0),
]


def digest(a) -> str:
    if isinstance(a, (bytes, bytearray)):
        return hashlib.sha256(bytes(a)).hexdigest()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run_case(c: dict) -> dict:
    from semstream import codec as C, selection as S, transport as T
    from semstream.synth import make_clip
    from semstream.video import GoP, gop_psnr

    clip = make_clip(c["clip"], c["W"], c["H"], c["frames"], seed=c["seed"])
    cfg = C.CodecConfig()
    prev = None
    gops = []
    for k in range(clip.gop_count):
        g = clip.gop(k)
        s = c["scales"][k]
        work = g if s == 1 else C.scale_gop(g, s, "down")
        I, P = C.encode_gop(work, cfg)
        sim = S.token_similarity(P, I)
        drop = np.zeros(I.mask.shape, dtype=bool)
        if c["drop"] > 0.0:
            drop = S.build_drop_mask(sim, c["drop"])
            P = C.apply_token_mask(P, drop)
        wire = [p.to_bytes() for p in T.packetize_tokens(I, scale=s) + T.packetize_tokens(P, scale=s)]
        rng = np.random.default_rng(1000 * c["seed"] + k)
        lost = sorted(int(j) for j in np.flatnonzero(rng.random(len(wire)) < c["loss"]))
        recv = [T.parse_packet(d) for j, d in enumerate(wire) if j not in set(lost)]
        shape = I.values.shape
        ri = T.reassemble([p for p in recv if p.kind == "I"], shape, "I", gop_id=k,
                          frame_shape=I.frame_shape)
        rp = T.reassemble([p for p in recv if p.kind == "P"], shape, "P", gop_id=k,
                          frame_shape=I.frame_shape)
        rec = C.decode_gop(ri, rp, cfg)
        up = rec if s == 1 else C.scale_gop(rec, s, "up", crop=(c["H"], c["W"]))
        if prev is not None:
            up = C.blend_boundary(prev, up, 2)
        prev = up
        psnr_db, pooled = gop_psnr(g, up)
        gops.append(dict(
            scale=s,
            lost=lost,
            k_drop=int(drop.sum()),
            src=digest(np.stack([f.samples for f in g.frames])),
            work=digest(np.stack([f.samples for f in work.frames])),
            tok_i=digest(I.values),
            tok_p=digest(P.values),
            p_mask=digest(P.mask.astype(np.uint8)),
            sim=digest(sim.values),
            drop=digest(drop.astype(np.uint8)),
            wire=digest(b"".join(len(d).to_bytes(4, "big") + d for d in wire)),
            wire_first=wire[0].hex() if len(wire[0]) <= 600 else None,
            n_packets=len(wire),
            rows_received=[int(len([p for p in recv if p.kind == "I"])),
                           int(len([p for p in recv if p.kind == "P"]))],
            i_img=digest(rec.frames[0].samples),
            p_img=digest(rec.frames[1].samples),
            out=digest(np.stack([f.samples for f in up.frames])),
            psnr_db=psnr_db,
            mse=pooled,
        ))
    return dict(case=c, gops=gops)


def main() -> None:
    sys.path.insert(0, str(REF))
    import scipy
    out = dict(
        generator="tests/golden/make_golden.py (live reference /root/reference/pkg/src/semstream)",
        numpy=np.__version__, scipy=scipy.__version__,
        cases=[run_case(c) for c in CASES],
    )
    OUT.write_text(json.dumps(out, indent=1))
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
