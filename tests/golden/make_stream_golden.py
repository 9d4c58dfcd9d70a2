"""Generate tests/golden/stream_golden.json from the LIVE reference CLI.

Run in the build container only (needs /root/reference):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_stream_golden.py

Each case runs the reference's own `semstream encode` (cli.py:77-120) on a
synthetic clip spec, then `semstream decode` (cli.py:141-190) on the stream it
wrote, and records the SHA-256 / size of the stream file (SMST container,
cli.py:34-35,67-74), the metadata sidecar (video.py:217-230) and the decoded
raw-rgb24 video (video.py:139-143).  The GPU test
(tests/test_gpu_streamfile.py) re-encodes the same clips through
paper_2602_03529_b200.streamfile and must reproduce every byte.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
import tempfile
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "stream_golden.json"

CASES = [
    dict(name="nm96x64_s3_drop10_res", spec="synth:noisy-motion:96x64:27:seed=3", scale=3,
         drop_rate=0.10, residual=True, blend_width=2, theta=0.02),
    dict(name="ms100x70_s2_tail_nores", spec="synth:moving-square:100x70:20:seed=1", scale=2,
         drop_rate=0.0, residual=False, blend_width=2, theta=0.02),
    dict(name="sd128x96_s2_drop25_res_n3", spec="synth:static-detail:128x96:18:seed=2", scale=2,
         drop_rate=0.25, residual=True, blend_width=3, theta=0.03),
]


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def main() -> None:
    sys.path.insert(0, str(REF))
    from semstream import cli

    out = {"source": "reference semstream CLI encode/decode (cli.py:77-190)", "cases": []}
    with tempfile.TemporaryDirectory() as tmp:
        for c in CASES:
            stream = str(Path(tmp) / f"{c['name']}.smst")
            rgb = str(Path(tmp) / f"{c['name']}.rgb")
            enc = argparse.Namespace(input=c["spec"], width=None, height=None, format="raw-rgb24",
                                     output=stream, scale=c["scale"], fps=30.0,
                                     theta=c["theta"], drop_rate=c["drop_rate"],
                                     blend_width=c["blend_width"], no_residual=not c["residual"])
            cli.cmd_encode(enc)
            dec = argparse.Namespace(input=stream, output=rgb, reference=None, format="raw-rgb24")
            cli.cmd_decode(dec)
            data = Path(stream).read_bytes()
            meta = Path(stream + ".meta.json").read_text()
            video = Path(rgb).read_bytes()
            out["cases"].append(dict(c, stream_sha256=sha(data), stream_bytes=len(data),
                                     meta_json=meta, video_sha256=sha(video),
                                     video_bytes=len(video)))
    OUT.write_text(json.dumps(out, indent=1) + "\n")
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
