"""Benchmark of the B200 codec hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one GoP (9 frames) of every stream on this GPU through the full
path: scale_gop(down) + encode_gop + token_similarity -> intelligent drop
(build_drop_mask + apply_token_mask, P layer) -> packetize (quantise, header,
mask, payload, CRC-32) -> parse + first-wins reassembly + mask-aware decode ->
scale_gop(up, crop) + blend_boundary, all 9 output frames materialised.

Workload (BASELINE.json configs[2]+[4]): S concurrent 1080p streams per GPU
(default 64), variable-resolution mode (half the streams at scale 3, half at
scale 2, pattern 3,3,2,2 per stream), 10% intelligent P-token drop, blend
width 2.  Weak scaling: every rank runs its own S streams (stream ids
rank*S + i); no collective touches the data path.

`value` is device-resident throughput (inputs already in HBM; every step's
input is 14.3 GB at S=64, far larger than the 126 MB L2, so no flush is
needed).  `e2e` runs the same pipeline through the public batched API with
pinned HOST frames: H2D of the step's input, the sender's packets D2H and the
receiver's packets H2D (the network boundary), and D2H of the reconstructed
frames, all inside the timed region.

--impl reference times the reference algorithm's CPU implementation (the
oracle port, oracle/semstream_oracle.py -- the reference itself is numpy and
cannot travel to the GPU box) on the host cores, one GoP per worker process
per step, on the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "1080p encode+decode frames/sec per B200 (1/2/4/8 GPU); PSNR delta vs CPU ref"
UNIT = "frames/s"
GOP = 9
SCALE_PATTERN = (3, 3, 2, 2)     # per-stream GoP scale sequence (variable resolution)
FALLBACK_HBM_GBS = 6650.0        # /opt/skills/guides/B200_PROFILING.md fallback


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--streams", type=int, default=64,
                    help="streams per GPU (--scaling weak) or in total (--scaling strong)")
    ap.add_argument("--scaling", choices=("weak", "strong"), default="weak",
                    help="weak: every GPU codes --streams streams (ids rank*S+i); strong: "
                         "--streams streams in total, stream_id %% N == rank (BASELINE configs[4])")
    ap.add_argument("--selftest-launcher", action="store_true",
                    help="CPU test hook: run the N-rank launch / sharding / max-over-ranks / "
                         "reporting path over gloo without GPU work")
    ap.add_argument("--lanes", type=int, default=2,
                    help="independent StreamBanks, each on its own CUDA stream (even)")
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--drop", type=float, default=0.10)
    ap.add_argument("--e2e-streams", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-workers", type=int, default=0, help="0 = auto")
    ap.add_argument("--no-rgb24", action="store_true",
                    help="skip the raw-rgb24 leg (uint8 frames in and out, SURVEY §8(d) variant)")
    ap.add_argument("--no-learned", action="store_true",
                    help="skip the learned-tokenizer leg (SURVEY f4, tensor-core path)")
    ap.add_argument("--no-learned-bf16", action="store_true",
                    help="skip the bf16 learned-tokenizer leg (the int8 leg still runs)")
    ap.add_argument("--learned-gops", type=int, default=32)
    ap.add_argument("--learned-lanes", type=int, default=1)
    ap.add_argument("--roofline-steps", type=int, default=3,
                    help="extra serialised steps timing each kernel alone")
    return ap.parse_args()


def workload_config(a) -> dict:
    per = "per GPU" if a.scaling == "weak" else "in total, sharded stream_id % N"
    return {
        "workload": f"{a.streams} concurrent {a.height}p streams {per}, variable-resolution "
                    f"(scales {SCALE_PATTERN} per stream, half the streams at each scale), "
                    f"{int(a.drop * 100)}% intelligent P-token drop, blend n=2, no network loss",
        "streams": a.streams,
        "streams_are": "per GPU" if a.scaling == "weak" else "total",
        "frame": [a.height, a.width, 3],
        "frame_dtype": "float32 in / float32 out (reference Frame dtype)",
        "gop_frames": GOP,
        "drop_rate": a.drop,
        "blend_width": 2,
        "l2": (f"inputs larger than L2: each step reads a fresh "
               f"{a.streams * GOP * a.height * a.width * 12 / 1e9:.1f} GB GoP batch "
               f"({a.streams} streams) vs the 126 MB L2"),
    }


# ---------------------------------------------------------------------------
# helpers

def scale_of(stream: int, k: int) -> int:
    half = 0 if stream % 2 == 0 else 2          # odd streams run the pattern shifted by 2 GoPs
    return SCALE_PATTERN[(k + half) % len(SCALE_PATTERN)]


_CLOCK_POLL = r"""
import sys, time, pynvml
pynvml.nvmlInit()
uuid = sys.argv[1]
try:
    h = pynvml.nvmlDeviceGetHandleByUUID(uuid)
except Exception:
    h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[2]))
get = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
    pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
print("max", pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM), flush=True)
while True:
    print(time.monotonic(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), int(get(h)),
          flush=True)
    time.sleep(0.002)
"""


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled through NVML every
    ~2 ms during the timed region, from a separate PROCESS (a thread of this
    one competes with the launch loop for the GIL and sampled only a few
    times per run).  Samples taken before the region opens are discarded."""

    BITS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
            0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.max_mhz = None
        self.err = ""
        self._p = None
        self._lines = []
        self._t = None
        self._t0 = None
        self._t1 = None

    def __enter__(self):
        import subprocess
        try:
            import torch
            uuid = str(torch.cuda.get_device_properties(self.index).uuid)
            uuid = uuid if uuid.startswith("GPU-") else f"GPU-{uuid}"
            self._p = subprocess.Popen([sys.executable, "-c", _CLOCK_POLL, uuid, str(self.index)],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                       text=True)
            first = self._p.stdout.readline().split()          # wait until polling runs
            if first and first[0] == "max":
                self.max_mhz = int(first[1])

            def reader():                       # drain the pipe; filter by the poller's clock
                for ln in self._p.stdout:
                    self._lines.append(ln)
            self._t = threading.Thread(target=reader, daemon=True)
            self._t.start()
            self._t0 = time.monotonic()             # CLOCK_MONOTONIC: shared with the poller
        except Exception as e:
            self.err = f"{type(e).__name__}: {e}"
        return self

    def __exit__(self, *exc):
        t1 = time.monotonic()
        if self._p is not None:
            time.sleep(0.01)
            self._p.kill()
            self._p.wait()
            if self._t is not None:
                self._t.join(timeout=2)
        for ln in list(self._lines):
            parts = ln.split()
            if len(parts) == 3 and self._t0 <= float(parts[0]) <= t1:
                self.samples.append((int(parts[1]), int(parts[2])))

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"],
                    "error": self.err}
        reasons = sorted({name for _, r in self.samples for bit, name in self.BITS.items()
                          if r & bit})
        return {"sm_mhz": statistics.median(m for m, _ in self.samples),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples),
                "source": "NVML, ~2 ms polling from a separate process inside the timed region"}


def measured_hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram bytes per launch of the dominant kernels from the committed ncu
    --set full capture (profiles/*_traffic.json), or None."""
    best = None
    for p in sorted((ROOT / "profiles").glob("*_traffic.json")):
        try:
            best = json.loads(p.read_text())
        except Exception:
            pass
    return best


# ---------------------------------------------------------------------------
# device input generation (synthetic clips of the named shape)

def make_inputs(stream_ids, H, W, device, n_sets=2):
    """[n_sets][n_streams, 9, H, W, 3] float32: per stream a textured square
    moving over a gradient (moving-square style) plus per-frame noise on odd
    streams (noisy-motion style); every stream has its own seed."""
    import torch
    n_streams = len(stream_ids)
    sets = []
    yy = torch.linspace(0, 1, H, device=device)[:, None]
    xx = torch.linspace(0, 1, W, device=device)[None, :]
    base = torch.stack([(0.25 + 0.5 * xx).expand(H, W), (0.25 + 0.5 * yy).expand(H, W),
                        torch.full((H, W), 0.4, device=device)], dim=-1)
    side = max(8, min(H, W) // 4)
    for k in range(n_sets):
        frames = torch.empty((n_streams, GOP, H, W, 3), dtype=torch.float32, device=device)
        for i, sid in enumerate(stream_ids):
            g = torch.Generator(device=device)
            g.manual_seed(1000 + sid)
            tex = torch.rand((side // 4 + 1, side // 4 + 1, 3), generator=g, device=device)
            tex = tex.repeat_interleave(4, 0).repeat_interleave(4, 1)[:side, :side]
            for t in range(GOP):
                idx = k * GOP + t
                img = base.clone()
                x = (4 * idx + 37 * sid) % max(W - side, 1)
                y = (2 * idx + 11 * sid) % max(H - side, 1)
                img[y:y + side, x:x + side] = tex
                if sid % 2:
                    img = img + 0.15 * (torch.rand((H, W, 3), generator=g, device=device) - 0.5)
                frames[i, t] = img.clamp_(0.0, 1.0)
        sets.append(frames)
    return sets


# ---------------------------------------------------------------------------
# our arm

def _coll_device(dev):
    """Collectives run on the GPU under NCCL, on host tensors under gloo (the
    SST_BENCH_SHARE_GPU hook and the CPU launcher self-test)."""
    import torch.distributed as dist
    return dev if dist.get_backend() == "nccl" else "cpu"


def max_over_ranks(ms: float, dev) -> float:
    """Device-timed step time, max over ranks (paper_2602_03529_b200.shard)."""
    from paper_2602_03529_b200.shard import max_over_ranks as _max
    return _max(ms, _coll_device(dev))


def gather_ranks(values, dev) -> list:
    """Every rank's small float vector (per-rank timing / stream counts), for
    the report only -- no collective touches the data path."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [list(values)]
    t = torch.tensor(list(values), dtype=torch.float64, device=_coll_device(dev))
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [[float(v) for v in o.cpu()] for o in out]


def my_streams(a, rank: int, world: int, per: int | None = None) -> list:
    """This rank's stream ids: weak scaling = its own
    ``per`` streams (rank*per + i), strong = stream_id % world == rank out of
    ``per`` in total."""
    from paper_2602_03529_b200.shard import rank_streams, strong_streams
    per = a.streams if per is None else per
    if a.scaling == "weak":
        return rank_streams(rank, world, per)
    if per < world:
        raise SystemExit(f"--scaling strong needs at least one stream per rank ({per} < {world})")
    return strong_streams(rank, world, per)


def total_streams(a, world: int, per: int | None = None) -> int:
    per = a.streams if per is None else per
    return per * world if a.scaling == "weak" else per


def to_rgb24(frames):
    """write_raw_video's bytes of float32 frames (video.py:139-143), on the device."""
    import torch
    return torch.round(frames * 255.0).to(torch.uint8)   # float32 product, half to even


def run_ours(a, rank, world, local_rank, rgb24: bool = False):
    """The bench workload through StreamBank.  rgb24: the same streams as
    raw-rgb24 bytes in and out (the reference CLI's file formats, cli.py:52-61
    and 181; the kernels fuse load_raw_video's q/255 and write_raw_video's
    quantiser)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2602_03529_b200.pipeline import StageTimer, StreamBank

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    mine = my_streams(a, rank, world)
    S, H, W = len(mine), a.height, a.width
    # Two lanes of streams: the even-phase streams and the odd-phase streams
    # (their scale patterns are offset by two GoPs, so at every step one lane
    # codes at s=3 and the other at s=2).  Each lane is an independent
    # StreamBank on its own CUDA stream: no dependency crosses lanes, so one
    # lane's latency-bound middle kernels overlap the other's HBM-bound
    # encode / reconstruction, and lanes are only joined at the end.  The
    # phase alternates over the rank's own streams, so every GPU codes half
    # of its streams at each scale in either scaling mode.
    even = [i for i in range(S) if i % 2 == 0]
    odd = [i for i in range(S) if i % 2 == 1]
    ne = len(even)
    inputs = make_inputs([mine[i] for i in even + odd], H, W, dev)
    if rgb24:
        inputs = [to_rgb24(x) for x in inputs]
        torch.cuda.empty_cache()
    out = torch.empty_like(inputs[0])
    lanes = []
    per = max(1, a.lanes // 2)                  # lanes per phase
    for phase, (lo, hi) in enumerate(((0, ne), (ne, S))):
        cuts = [lo + (hi - lo) * j // per for j in range(per + 1)]
        for j in range(per):
            if cuts[j + 1] > cuts[j]:
                lanes.append(dict(sl=slice(cuts[j], cuts[j + 1]), phase=phase,
                                  n=cuts[j + 1] - cuts[j]))
    fused = not rgb24 and os.environ.get("SST_BENCH_FUSED", "0") == "1"
    for ln in lanes:
        ln["bank"] = StreamBank(ln["n"], H, W, concurrent_groups=False, fused=fused)
        ln["stream"] = torch.cuda.Stream(device=dev)

    class _Banks:                       # aggregate view for launch counting / timers
        @property
        def launches(self):
            return sum(ln["bank"].launches for ln in lanes)

        def set_timer(self, t):
            for ln in lanes:
                ln["bank"].set_timer(t)
    bank = _Banks()

    def groups(k):
        fr = inputs[k % 2]
        out_g = {}
        for ln in lanes:
            s = scale_of(ln["phase"], k)
            out_g[s] = (fr[ln["sl"]], out[ln["sl"]])
        return ({s: v[0] for s, v in out_g.items()}, {s: v[1] for s, v in out_g.items()}, None)

    def one_step(k):
        main = torch.cuda.current_stream()
        fr = inputs[k % 2]
        for ln in lanes:
            st = ln["stream"]
            if k == 0:
                st.wait_stream(main)
            s = scale_of(ln["phase"], k)
            with torch.cuda.stream(st):
                ln["bank"].step({s: fr[ln["sl"]]}, {s: out[ln["sl"]]}, {s: list(range(ln["n"]))},
                                {s: [k] * ln["n"]}, drop_rate=a.drop)

    def join():
        main = torch.cuda.current_stream()
        for ln in lanes:
            main.wait_stream(ln["stream"])

    for k in range(a.warmup):
        one_step(k)
    join()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = bank.launches
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        torch.cuda.synchronize()
        t_start.record()
        for ln in lanes:
            ln["stream"].wait_stream(torch.cuda.current_stream())
        for k in range(a.warmup, a.warmup + a.steps):
            one_step(k)
        join()
        t_end.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = t_start.elapsed_time(t_end)
    ms_max = ms
    if world > 1:
        ms_max = max_over_ranks(ms, dev)
    per_rank = gather_ranks([ms, S], dev)
    launches = bank.launches - launches0
    # Per-kernel roofline: a few extra steps with the lanes serialised on one
    # stream so that every kernel's CUDA-event duration is its own (in the
    # timed run the two lanes overlap and each kernel shares the HBM).
    timer = StageTimer(lead_cycles=2_000_000)     # ~1 ms spin ahead of every stage
    bank.set_timer(timer)
    for k in range(a.warmup + a.steps, a.warmup + a.steps + a.roofline_steps):
        fr = inputs[k % 2]
        for ln in lanes:
            s = scale_of(ln["phase"], k)
            ln["bank"].step({s: fr[ln["sl"]]}, {s: out[ln["sl"]]}, {s: list(range(ln["n"]))},
                            {s: [k] * ln["n"]}, drop_rate=a.drop)
    torch.cuda.synchronize()
    bank.set_timer(None)
    stages = timer.summary()
    frames_total = total_streams(a, world) * GOP * a.steps
    assert frames_total == sum(int(n) for _, n in per_rank) * GOP * a.steps
    value = frames_total / (ms_max / 1000.0)

    # quality of one GoP per scale vs the source (device metric)
    psnr = {}
    fr, ou, ids = groups(a.warmup + a.steps - 1)
    for s, o in ou.items():
        src = fr[s][0]
        sc = 1.0 / 255.0 if rgb24 else 1.0
        mse = (((o[0].double() - src.double()) * sc) ** 2).mean().item()
        psnr[f"s{s}"] = 99.0 if mse <= 0 else min(99.0, 10 * np.log10(1.0 / mse))

    res = dict(ms=ms_max, value=value, stages=stages, launches=launches,
               clocks=clocks.summary(), psnr=psnr,
               per_rank=[{"rank": r, "streams": int(n), "ms": round(m, 3),
                          "frames_per_s": round(n * GOP * a.steps / (m / 1000.0), 1)}
                         for r, (m, n) in enumerate(per_rank)])
    res["roofline"] = roofline(a, stages, S // len(lanes), a.roofline_steps * len(lanes),
                               bpe=1 if rgb24 else 4)
    del inputs, out
    torch.cuda.empty_cache()
    if not a.no_e2e:
        res["e2e"] = run_e2e(a, rank, world, local_rank, rgb24=rgb24)
    return res


def rgb24_leg(a, rank, world, local_rank, dev) -> dict:
    """The bench workload over raw-rgb24 frames (uint8 in, uint8 out: the
    reference CLI's encode input and decode output, video.py:103-143), with a
    device-side parity check: the uint8 output of two streams x two GoPs
    equals write_raw_video's bytes of the float32 path's output on the same
    (converted) input, bit for bit."""
    import numpy as np
    import torch

    from paper_2602_03529_b200.pipeline import StreamBank
    res = run_ours(a, rank, world, local_rank, rgb24=True)
    out = {"workload": "as the headline, frames as raw-rgb24 bytes in and out "
                       "(uint8 [S][9][1080][1920][3]; load_raw_video's q/255 fused into K1, "
                       "write_raw_video's quantiser into K5)",
           "value": round(res["value"], 2), "unit": UNIT,
           "ms_per_step": round(res["ms"] / a.steps, 3), "gpu_launches": res["launches"],
           "stages": {k: {"ms_per_launch": round(v[0] / v[1], 4), "launches": v[1]}
                      for k, v in res["stages"].items()},
           "roofline": res["roofline"], "path_roofline": path_roofline(a, res["value"] / world, bpe=1),
           "clocks": res["clocks"], "psnr_db_vs_u8_source": res["psnr"], "e2e": res.get("e2e")}
    # parity: uint8 path vs the float32 path + write_raw_video's quantiser
    H, W = a.height, a.width
    src = to_rgb24(make_inputs([0, 1], H, W, dev, n_sets=2)[0])
    b8, bf = StreamBank(2, H, W), StreamBank(2, H, W)
    # load_raw_video's float32(q) / 255, correctly rounded (numpy; torch's
    # CUDA division by a scalar multiplies by the reciprocal)
    q255 = torch.from_numpy(np.arange(256, dtype=np.float32) / np.float32(255.0)).to(dev)
    ok = True
    for k, s in enumerate((3, 2)):
        fr8 = src
        frf = q255[src.long()]
        o8, of = torch.empty_like(fr8), torch.empty_like(frf)
        b8.step({s: fr8}, {s: o8}, {s: [0, 1]}, {s: [k, k]}, drop_rate=a.drop)
        bf.step({s: frf}, {s: of}, {s: [0, 1]}, {s: [k, k]}, drop_rate=a.drop)
        torch.cuda.synchronize()
        ok = ok and bool(torch.equal(o8, to_rgb24(of)))
    out["parity"] = {"sample": "2 streams x 2 GoPs (s=3 then s=2, blend n=2), 10% drop",
                     "uint8_equals_quantised_float32_path": ok,
                     "tests": "tests/test_gpu_rgb24.py (vs the oracle and the reference's own "
                              "load_raw_video / write_raw_video)"}
    return out


def roofline(a, stages, gops_per_launch, _launches_hint=None, bpe: int = 4) -> dict:
    """Achieved GB/s of the dominant kernel: algorithmic bytes per launch /
    average CUDA-event launch duration inside the timed region (bpe: bytes
    per frame sample, 4 = float32, 1 = raw-rgb24)."""
    H, W = a.height, a.width
    frame_bytes = H * W * 3 * bpe
    # per GoP (one stream): K1 reads 9 frames + writes tokens/sim;
    # K5 writes 9 frames + reads the two working images (+ the previous P image)
    def tokens_bytes(s):
        h, w = -(-H // s), -(-W // s)
        ht, wt = -(-h // 8), -(-w // 8)
        return ht * wt * (2 * 12 * 8 + 8), 3 * h * w * 3 * 4
    avg_tok = sum(tokens_bytes(s)[0] for s in (2, 3)) / 2
    avg_img = sum(tokens_bytes(s)[1] for s in (2, 3)) / 2
    per_gop = {"K1_encode": GOP * frame_bytes + avg_tok,
               "K5_upscale_blend": GOP * frame_bytes + avg_img}
    peak, peak_src = measured_hbm_peak()
    best = None
    for name, bytes_gop in per_gop.items():
        if name not in stages:
            continue
        tot_ms, launches = stages[name]
        algo = bytes_gop * gops_per_launch
        avg_s = tot_ms / launches / 1000.0
        ach = algo / avg_s / 1e9
        cand = dict(kernel=name, bound="hbm", achieved=round(ach, 1), peak=peak, unit="GB/s",
                    frac=round(ach / peak, 4), peak_source=peak_src,
                    algorithmic_bytes_per_launch=int(algo),
                    avg_launch_ms=round(avg_s * 1000, 4))
        if best is None or tot_ms > best["_tot"]:
            best = dict(cand, _tot=tot_ms)
    if best is None:
        return None
    best.pop("_tot")
    tr = ncu_traffic()
    best["traffic"] = None
    if tr and best["kernel"] in tr and bpe == 4:
        # ncu --set full DRAM bytes per GoP x GoPs per launch of this run
        best["traffic"] = int(tr[best["kernel"]] * gops_per_launch)
        best["traffic_source"] = tr.get("_source")
    return best


def path_roofline(a, fps, bpe: int = 4) -> dict:
    """Whole path against HBM: SURVEY §8(d) algorithmic bytes per frame
    (read the frame once, write it once, fp32 -- or raw-rgb24 bytes -- +
    packets) x frames/s."""
    peak, src = measured_hbm_peak()
    per_frame = a.height * a.width * 3 * (bpe + bpe)
    ach = per_frame * fps / 1e9
    return {"bytes_per_frame": per_frame, "achieved": round(ach, 1), "peak": peak,
            "unit": "GB/s", "frac": round(ach / peak, 4),
            "roofline_fps": round(peak * 1e9 / per_frame, 1)}


def run_e2e(a, rank, world, local_rank, rgb24: bool = False) -> dict:
    """Same pipeline through the public batched API with pinned host buffers:
    frames H2D -> sender (K1-K3) -> packets D2H -> packets H2D -> receiver
    (K4, K5) -> frames D2H, every step, inside the timed region.  The streams
    are split over `lanes` independent StreamBanks, each on its own CUDA
    stream, so one lane's H2D overlaps another's kernels and D2H (PCIe is
    full duplex)."""
    import torch
    import torch.distributed as dist

    from paper_2602_03529_b200.pipeline import StreamBank

    dev = torch.device("cuda", local_rank)
    mine = my_streams(a, rank, world, a.e2e_streams)
    E, H, W = len(mine), a.height, a.width
    lanes = max(1, min(int(os.environ.get("SST_E2E_LANES", "8")), E))   # one stream per lane
    per = [list(range(E))[i::lanes] for i in range(lanes)]
    src_dev = make_inputs(mine, H, W, dev, n_sets=1)[0]
    fdt, bpe = torch.float32, 4
    if rgb24:
        src_dev, fdt, bpe = to_rgb24(src_dev), torch.uint8, 1
    fshape = tuple(src_dev.shape[1:])
    L = []
    for ids in per:
        g = len(ids)
        bank = StreamBank(g, H, W)
        # pinned host frames of this lane's streams (one copy per lane only)
        h_in = torch.empty((g,) + fshape, dtype=fdt, pin_memory=True)
        h_in.copy_(src_dev[torch.tensor(ids, device=dev)])
        L.append(dict(
            ids=ids, bank=bank, stream=torch.cuda.Stream(device=dev),
            h_in=h_in, h_out=torch.empty((g,) + fshape, dtype=fdt, pin_memory=True),
            d_in=torch.empty((g,) + fshape, dtype=fdt, device=dev),
            d_out=torch.empty((g,) + fshape, dtype=fdt, device=dev),
            pk={s: torch.empty(c.arena.shape, dtype=torch.uint8).pin_memory()
                for s, c in bank.codecs.items()},
            ln={s: torch.empty(c.lengths.shape, dtype=torch.int32).pin_memory()
                for s, c in bank.codecs.items()}))
    del src_dev
    torch.cuda.empty_cache()
    counters = {"h2d": 0, "d2h": 0}

    def one(k):
        s = SCALE_PATTERN[k % len(SCALE_PATTERN)]
        for ln in L:
            bank, g = ln["bank"], len(ln["ids"])
            with torch.cuda.stream(ln["stream"]):
                c = bank.codecs[s]
                ln["d_in"].copy_(ln["h_in"], non_blocking=True)
                counters["h2d"] += ln["h_in"].numel() * bpe
                parity = bank.step_idx & 1
                c.set_gop_ids([k] * g)
                c.encode(ln["d_in"], g, c.drop_k(a.drop))
                npk = g * c.n_pkt_per_gop
                # sender -> wire (host memory) -> receiver
                ln["pk"][s][:npk].copy_(c.arena[:npk], non_blocking=True)
                ln["ln"][s][:npk].copy_(c.lengths[:npk], non_blocking=True)
                counters["d2h"] += npk * c.slot + npk * 4
                c.arena[:npk].copy_(ln["pk"][s][:npk], non_blocking=True)
                c.lengths[:npk].copy_(ln["ln"][s][:npk], non_blocking=True)
                counters["h2d"] += npk * c.slot + npk * 4
                c.decode(g, parity)
                staged = bank._prev_descs(s, list(range(g)))
                c.reconstruct(g, parity, ln["d_out"], None if staged is None else staged[0])
                if staged is not None:
                    bank.rings[s].release(staged[1])
                for i in range(g):
                    bank.last[i] = (s, parity, i)
                bank.step_idx += 1
                ln["h_out"].copy_(ln["d_out"], non_blocking=True)
                counters["d2h"] += ln["h_out"].numel() * bpe

    def sync_all():
        for ln in L:
            ln["stream"].synchronize()

    for k in range(a.warmup):
        one(k)
    sync_all()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    counters["h2d"] = counters["d2h"] = 0
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    main = torch.cuda.current_stream()
    wall0 = time.perf_counter()
    t0.record(main)
    for ln in L:
        ln["stream"].wait_stream(main)
    for k in range(a.warmup, a.warmup + a.steps):
        one(k)
    for ln in L:
        main.wait_stream(ln["stream"])
    t1.record(main)
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    ms = t0.elapsed_time(t1)
    if world > 1:
        ms = max_over_ranks(ms, dev)
    frames = total_streams(a, world, a.e2e_streams) * GOP * a.steps
    return {"value": round(frames / (ms / 1000.0), 2), "unit": UNIT,
            "h2d_bytes_per_step": int(counters["h2d"] // a.steps),
            "d2h_bytes_per_step": int(counters["d2h"] // a.steps),
            "streams": total_streams(a, world, a.e2e_streams), "streams_this_rank": E,
            "lanes": lanes, "wall_s": round(wall, 3),
            "path": f"StreamBank public API on pinned host {'raw-rgb24' if rgb24 else 'float32'} "
                    "frames: frames H2D, packets D2H + H2D (network boundary), frames D2H, all "
                    f"inside the timed region; {lanes} CUDA-stream lanes overlap PCIe "
                    "directions with compute"}


# ---------------------------------------------------------------------------
# CPU reference: the UNMODIFIED reference package installed in baseline/_ref
# (python -m pip install --no-index --no-build-isolation --no-deps --target
# baseline/_ref <copy of /root/reference/pkg>; git-ignored, travels with the
# snapshot) run through its own public API; the oracle port only when that
# install is absent.

REF_DIR = ROOT / "baseline" / "_ref"


def reference_kind() -> str:
    return "reference" if (REF_DIR / "semstream" / "__init__.py").is_file() else "port"


def _init_worker():
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))


_CLIP_CACHE: dict = {}
_PREV_OUT: dict = {}


def _ref_gop(H, W, sid, k, s, drop):
    """One GoP through the stock reference composition (session.py:134-170
    sender, 323-348 receiver, without the emulated network): scale_gop(down)
    -> encode_gop -> token_similarity -> build_drop_mask -> apply_token_mask
    -> packetize_tokens -> to_bytes -> parse_packet -> reassemble x2 ->
    decode_gop -> scale_gop(up, crop) -> blend_boundary(n=2) against the
    worker's previous output.  Returns (compute seconds, PSNR dB)."""
    from semstream import codec, selection, synth, transport, video
    key = ("ref", H, W, sid, k)
    if key not in _CLIP_CACHE:          # clip generation is not part of the timed work
        name = "moving-square" if sid % 2 == 0 else "noisy-motion"
        _CLIP_CACHE.clear()
        _CLIP_CACHE[key] = synth.make_clip(name, W, H, GOP * (k + 1), seed=sid).gop(k)
    gop = _CLIP_CACHE[key]
    t0 = time.perf_counter()
    cfg = codec.CodecConfig()
    working = codec.scale_gop(gop, s, "down")
    i_tok, p_tok = codec.encode_gop(working, cfg)
    if drop > 0.0:
        sim = selection.token_similarity(p_tok, i_tok)
        p_tok = codec.apply_token_mask(p_tok, selection.build_drop_mask(sim, drop))
    wire = [p.to_bytes() for p in transport.packetize_tokens(i_tok, scale=s)
            + transport.packetize_tokens(p_tok, scale=s)]
    parsed = [transport.parse_packet(d) for d in wire]
    shape = i_tok.values.shape
    ri = transport.reassemble([p for p in parsed if p.kind == "I"], shape, "I", gop_id=k,
                              frame_shape=i_tok.frame_shape)
    rp = transport.reassemble([p for p in parsed if p.kind == "P"], shape, "P", gop_id=k,
                              frame_shape=i_tok.frame_shape)
    recon = codec.scale_gop(codec.decode_gop(ri, rp, cfg), s, "up", crop=(H, W))
    prev = _PREV_OUT.get((H, W))
    if prev is not None:
        recon = codec.blend_boundary(prev, recon, 2)
    dt = time.perf_counter() - t0
    _PREV_OUT[(H, W)] = recon
    return dt, video.gop_psnr(gop, recon)[0]


def _port_gop(H, W, sid, k, s, drop):
    from oracle import semstream_oracle as O
    from oracle.synth import make_clip
    key = ("port", H, W, sid, k)
    if key not in _CLIP_CACHE:
        name = "moving-square" if sid % 2 == 0 else "noisy-motion"
        _CLIP_CACHE.clear()
        _CLIP_CACHE[key] = make_clip(name, W, H, GOP * (k + 1), seed=sid).gop(k)
    frames = _CLIP_CACHE[key]
    t0 = time.perf_counter()
    res = O.pipeline_gop(frames, s, gop_id=k, drop_rate=drop, prev_out=_PREV_OUT.get((H, W)))
    dt = time.perf_counter() - t0
    _PREV_OUT[(H, W)] = res["frames"]
    return dt, O.gop_psnr(list(frames), res["frames"])[0]


def _cpu_worker(job):
    H, W, sid, k, s, drop, kind = job
    return (_ref_gop if kind == "reference" else _port_gop)(H, W, sid, k, s, drop)


def host_info() -> dict:
    """What the CPU arm ran on (nproc, CPU model, library versions)."""
    info = {"nproc": os.cpu_count()}
    try:
        info["affinity_cores"] = len(os.sched_getaffinity(0))
    except Exception:
        pass
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                info["cpu_model"] = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    try:
        import numpy
        import scipy
        info["numpy"], info["scipy"] = numpy.__version__, scipy.__version__
    except Exception:
        pass
    try:
        import psutil
        info["mem_available_gb"] = round(psutil.virtual_memory().available / 1e9, 1)
    except Exception:
        pass
    info["python"] = sys.version.split()[0]
    return info


def cpu_workers(a) -> tuple:
    """(workers, why): every host core the process may use, capped only by
    memory (~1.2 GB peak RSS per 1080p GoP worker, measured: 0.66 GB for the
    reference pipeline plus the cached clip) and 128."""
    if a.cpu_workers:
        return a.cpu_workers, "--cpu-workers"
    try:
        n = len(os.sched_getaffinity(0))
    except Exception:
        n = os.cpu_count() or 1
    why = "all host cores"
    try:
        import psutil
        per = 1.2e9 * (a.height * a.width) / (1080 * 1920)
        cap = max(1, int(psutil.virtual_memory().available // max(per, 1e8)))
        if cap < n:
            n, why = cap, f"memory cap ({per / 1e9:.1f} GB per worker)"
    except Exception:
        pass
    if n > 128:
        n, why = 128, "capped at 128"
    return max(1, n), why


def cpu_sample(a, steps: int, warm: int = 0, kind: str | None = None):
    """`steps` timed rounds of one GoP per worker process (pool wall clock per
    round, clip generation excluded: every worker's clip is materialised by an
    untimed round first).  Returns (workers, why, kind, round walls, psnrs)."""
    import multiprocessing as mp
    kind = kind or reference_kind()
    n, why = cpu_workers(a)
    ctx = mp.get_context("spawn")
    walls, psnrs = [], []
    with ctx.Pool(n, initializer=_init_worker) as pool:
        pool.map(_cpu_worker, [(a.height, a.width, i, 0, scale_of(i, 0), a.drop, kind)
                               for i in range(n)], chunksize=1)
        for r in range(warm + steps):
            jobs = [(a.height, a.width, i, 0, scale_of(i, r), a.drop, kind) for i in range(n)]
            t0 = time.perf_counter()
            out = pool.map(_cpu_worker, jobs, chunksize=1)
            wall = time.perf_counter() - t0
            if r >= warm:
                walls.append(wall)
                psnrs.extend(p for _, p in out)
    return n, why, kind, walls, psnrs


def _cpu_record(a, n, why, kind, walls) -> dict:
    what = ("the unmodified reference package (baseline/_ref semstream, its public API)"
            if kind == "reference" else "oracle/semstream_oracle.py (port; baseline/_ref absent)")
    return {"value": round(n * GOP * len(walls) / sum(walls), 3), "unit": UNIT, "cores": n,
            "kind": kind, "workers_why": why, "host": host_info(),
            "sample": f"{len(walls)} round(s) x {n} worker processes x one {a.height}p GoP each "
                      f"(9 frames, scales {sorted({scale_of(i, 0) for i in range(n)})}, "
                      f"{int(a.drop * 100)}% drop, blend n=2), {what}; throughput from the "
                      f"pool's wall clock per round ({sum(walls):.1f} s total), one thread per "
                      f"worker (OMP/OPENBLAS/MKL_NUM_THREADS=1)"}


def run_reference(a) -> dict:
    n, why, kind, walls, psnrs = cpu_sample(a, a.steps, a.warmup)
    rec = _cpu_record(a, n, why, kind, walls)
    return dict(value=rec["value"], ms=1000 * sum(walls) / len(walls), record=rec,
                psnr=statistics.mean(psnrs))


def cpu_baseline(a) -> dict:
    n, why, kind, walls, _ = cpu_sample(a, 1, 1)
    return _cpu_record(a, n, why, kind, walls)


def single_stream_latency(a, device) -> dict:
    """Real-time view (north_star: >= 30 fps per 1080p stream): ONE stream,
    one GoP at a time (each GoP blends with the previous one), variable scale
    3,3,2,2; device time per GoP (encode .. reconstruct, 9 frames) with the
    GoP resident in HBM -- eager (StreamBank) and with every step replayed as
    a CUDA graph (GraphedStreamBank) -- and the frame rate that implies."""
    import torch
    from paper_2602_03529_b200.pipeline import GraphedStreamBank, StreamBank
    H, W = a.height, a.width
    fr = make_inputs([0], H, W, device, n_sets=1)[0]
    out = torch.empty_like(fr)
    n, warm = 24, 4

    def timed(run):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(n)]
        walls = []
        for k in range(warm + n):
            s = SCALE_PATTERN[k % len(SCALE_PATTERN)]
            t0 = time.perf_counter()
            if k >= warm:
                ev[k - warm][0].record()
            run(k, s)
            if k >= warm:
                ev[k - warm][1].record()
            torch.cuda.synchronize()          # one GoP in flight: latency, not throughput
            if k >= warm:
                walls.append((time.perf_counter() - t0) * 1e3)
        ms = sorted(b.elapsed_time(e) for b, e in ev)
        walls.sort()
        return ms, walls

    bank = StreamBank(1, H, W)
    eager, eager_w = timed(lambda k, s: bank.step({s: fr}, {s: out}, {s: [0]}, {s: [k]},
                                                  drop_rate=a.drop))
    gbank = GraphedStreamBank(H, W, fr, out, drop_rate=a.drop)
    graph, graph_w = timed(lambda k, s: gbank.step(s, k))
    med = graph[len(graph) // 2]
    return {"stream": f"1 x {H}p, scales {SCALE_PATTERN}, {int(a.drop * 100)}% drop, blend n=2",
            "gop_ms_median": round(med, 3), "gop_ms_max": round(graph[-1], 3),
            "path": "GraphedStreamBank (each step one CUDA-graph replay, 14 kernels)",
            "eager_gop_ms_median": round(eager[len(eager) // 2], 3),
            "frames_per_s_single_stream": round(GOP / med * 1e3, 1),
            "realtime_30fps_budget_ms_per_gop": round(GOP / 30 * 1e3, 1),
            "host_wall_ms_per_gop": {"eager": round(eager_w[len(eager_w) // 2], 3),
                                     "graph": round(graph_w[len(graph_w) // 2], 3)}}


def loss_legs(a, device) -> dict:
    """BASELINE.json configs[3]: 1080p, s=3, 32 GoPs per
    launch with (a) intelligent P-token dropping at 10 % / 30 % and (b) seeded
    Bernoulli packet loss at 10 % / 30 % on the I+P packet list, decoder
    zero-fill + I-block concealment.  Device-resident frames/s, and for GoP 0
    the PSNR of the GPU reconstruction vs the CPU reference algorithm on the
    same lost-packet set (bit-exact expected)."""
    import numpy as np
    import torch

    from oracle import semstream_oracle as O
    from paper_2602_03529_b200.pipeline import GopCodec
    from paper_2602_03529_b200.video import gop_psnr_device
    H, W, s, G = a.height, a.width, 3, 32
    frames = make_inputs(list(range(G)), H, W, device, n_sets=1)[0]
    out = torch.empty_like(frames)
    codec = GopCodec(G, H, W, s)
    codec.set_gop_ids([0] * G)
    npk = codec.n_pkt_per_gop
    res = {}
    for kind, rate in (("drop", 0.10), ("drop", 0.30), ("loss", 0.10), ("loss", 0.30)):
        drop_k = codec.drop_k(rate) if kind == "drop" else 0
        present, lost0 = None, None
        if kind == "loss":
            rng = np.random.default_rng(int(rate * 100))
            keep = (rng.random(G * npk) >= rate).astype(np.uint8)
            present = torch.from_numpy(keep).to(device)
            lost0 = set(int(j) for j in np.flatnonzero(keep[:npk] == 0))

        def step():
            codec.encode(frames, G, drop_k)
            codec.decode(G, 0, present=present)
            codec.reconstruct(G, 0, out)

        for _ in range(2):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 5
        e0.record()
        for _ in range(n):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        src = frames[0].cpu().numpy()
        ref = O.pipeline_gop(src, s, gop_id=0, drop_rate=rate if kind == "drop" else 0.0,
                             lost=lost0)
        gpu = out[0].cpu().numpy()
        p_gpu, _ = gop_psnr_device(frames[0], out[0])          # GPU metric kernel
        p_ref, _ = O.gop_psnr(list(src), list(ref["frames"]))
        res[f"{kind}_{int(rate * 100)}pct"] = {
            "frames_per_s": round(G * GOP / ms * 1e3, 1),
            "psnr_gpu_db": round(p_gpu, 4), "psnr_cpu_ref_db": round(p_ref, 4),
            "bit_exact": bool(np.array_equal(gpu, np.stack(ref["frames"])))}
    return {"workload": f"{G} x {H}p GoPs per launch, s=3, no blending (first GoP of each "
                        "stream); drop = intelligent P-token dropping, loss = Bernoulli packet "
                        "loss with zero-fill + I concealment", **res}


def small_configs(a, device) -> dict:
    """BASELINE.json configs[0] and configs[1] on the GPU:
    [0] the 17-frame 256x256 clip (2 GoPs, the last one tail-padded) through
        the learned tokenizer (random-init weights, encode -> FSQ -> packetise
        -> decode -> upscale, tcgen05) at s=2, and through the reference proxy
        path at s=2 (bit-exact vs the CPU reference);
    [1] a 720p 33-frame clip (4 GoPs) through the proxy path, no loss:
        frames/s for 64 such streams per launch (device-resident) and GoP-0
        parity."""
    import numpy as np
    import torch

    from oracle import learned_i8_oracle as LO8
    from oracle import semstream_oracle as O
    from oracle.synth import make_clip
    from paper_2602_03529_b200.learned_i8 import LearnedI8Config, LearnedI8GopCodec
    from paper_2602_03529_b200.pipeline import GopCodec, StreamBank

    out = {}
    # ---- configs[0]
    clip = make_clip("moving-square", 256, 256, 17, seed=0)
    gops = np.stack([clip.gop(0), clip.gop(1)])
    fr = torch.from_numpy(gops).to(device)
    lc = LearnedI8GopCodec(2, 256, 256, 2, cfg=LearnedI8Config())
    o = torch.empty_like(fr)
    lc.set_gop_ids([0, 1])
    for _ in range(3):
        lc.step(fr, o, 2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        lc.step(fr, o, 2)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    codes, idx, mask, hw = lc.model.encode_frames(fr, 2)
    oc, oi, _ = LO8.encode(gops, 2, lc.model.host_weights)
    agree = float((idx.cpu().numpy() == oi).mean())
    dec = lc.model.decode_tokens(codes, mask, hw).cpu().numpy()
    dec_exact = bool(np.array_equal(dec, LO8.decode(oc, np.ones(oc.shape[:-1], np.uint8), hw,
                                                    lc.model.host_weights)))
    bank = StreamBank(1, 256, 256)
    po = torch.empty_like(fr[:1])
    prev, exact = None, True
    for k in range(2):
        bank.step({2: fr[k:k + 1].contiguous()}, {2: po}, {2: [0]}, {2: [k]})
        ref = O.pipeline_gop(gops[k], 2, gop_id=k, prev_out=prev)
        prev = ref["frames"]
        exact &= bool(np.array_equal(po[0].cpu().numpy(), np.stack(ref["frames"])))
    out["c0_tiny_256x256x17"] = {
        "learned_gop_ms": round(ms, 3),
        "learned_frames_per_s": round(17 / (ms / 1e3), 1),
        "learned_fsq_index_agreement_vs_oracle": round(agree, 5),
        "learned_decoded_frames_bit_exact_vs_oracle": dec_exact,
        "learned_model": "int8 (kind::i8), exact vs oracle/learned_i8_oracle.py",
        "proxy_s2_bit_exact_vs_cpu_reference": exact,
        "note": "one clip (2 GoPs per launch): launch-latency bound, not a throughput config"}
    # ---- configs[1]
    H, W, S = 720, 1280, 64
    frames = make_inputs(list(range(S)), H, W, device, n_sets=1)[0]
    res = {}
    for s in (2, 3):
        c = GopCodec(S, H, W, s)
        c.set_gop_ids([0] * S)
        o2 = torch.empty_like(frames)

        def step():
            c.encode(frames, S, 0)
            c.decode(S, 0)
            c.reconstruct(S, 0, o2)

        for _ in range(2):
            step()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        ref = O.pipeline_gop(frames[0].cpu().numpy(), s, gop_id=0)
        res[f"s{s}"] = {"frames_per_s": round(S * GOP / ms * 1e3, 1),
                        "bit_exact_gop0": bool(np.array_equal(o2[0].cpu().numpy(),
                                                              np.stack(ref["frames"])))}
    out["c1_720p_x64_streams"] = res
    return out


def cpu_reference_gop(src, s: int, drop: float, gop_id: int = 0):
    """(frames [9,H,W,3], psnr_db, kind): one GoP through the unmodified
    reference (baseline/_ref) when installed, else the oracle port; PSNR by
    the reference's own gop_psnr."""
    import numpy as np
    if reference_kind() == "reference":
        _init_worker()
        from semstream import codec, selection, transport, video
        gop = video.GoP(gop_id, tuple(video.Frame(f, timestamp_index=t) for t, f in enumerate(src)))
        cfg = codec.CodecConfig()
        working = codec.scale_gop(gop, s, "down")
        i_tok, p_tok = codec.encode_gop(working, cfg)
        if drop > 0.0:
            p_tok = codec.apply_token_mask(p_tok, selection.build_drop_mask(
                selection.token_similarity(p_tok, i_tok), drop))
        parsed = [transport.parse_packet(p.to_bytes()) for p in
                  transport.packetize_tokens(i_tok, scale=s) + transport.packetize_tokens(p_tok, scale=s)]
        sh = i_tok.values.shape
        ri = transport.reassemble([p for p in parsed if p.kind == "I"], sh, "I", gop_id=gop_id,
                                  frame_shape=i_tok.frame_shape)
        rp = transport.reassemble([p for p in parsed if p.kind == "P"], sh, "P", gop_id=gop_id,
                                  frame_shape=i_tok.frame_shape)
        rec = codec.scale_gop(codec.decode_gop(ri, rp, cfg), s, "up", crop=src.shape[1:3])
        return np.stack([f.samples for f in rec.frames]), video.gop_psnr(gop, rec)[0], "reference"
    from oracle import semstream_oracle as O
    frames = np.stack(O.pipeline_gop(src, s, gop_id=gop_id, drop_rate=drop)["frames"])
    return frames, O.gop_psnr(list(src), list(frames))[0], "port"


def parity_sample(a, device) -> dict:
    """PSNR delta vs the CPU reference on one full-size GoP: the same
    synthetic 1080p GoP through the GPU path (PSNR by the GPU metric kernel,
    csrc/metrics.cu) and through the reference (PSNR by its gop_psnr)."""
    import numpy as np
    import torch

    from oracle.synth import make_clip
    from paper_2602_03529_b200.pipeline import StreamBank
    from paper_2602_03529_b200.video import gop_psnr_device

    src = make_clip("moving-square", a.width, a.height, GOP, seed=0).gop(0)
    s = scale_of(0, 0)
    bank = StreamBank(1, a.height, a.width, concurrent_groups=False)
    fr = torch.from_numpy(src[None].copy()).to(device)
    out = torch.empty_like(fr)
    bank.step({s: fr}, {s: out}, {s: [0]}, {s: [0]}, drop_rate=a.drop)
    p_gpu, _ = gop_psnr_device(fr[0], out[0])
    gpu = out.cpu().numpy()[0]
    ref, p_ref, kind = cpu_reference_gop(src, s, a.drop)
    return {"sample": f"moving-square {a.height}p GoP, s={s}, {int(a.drop * 100)}% drop",
            "cpu_side": kind, "psnr_gpu_db": round(p_gpu, 6), "psnr_cpu_ref_db": round(p_ref, 6),
            "psnr_delta_db": p_gpu - p_ref,
            "max_abs_diff": float(np.abs(gpu.astype(np.float64) - ref).max()),
            "bit_exact": bool(np.array_equal(gpu, ref))}


def residual_leg(a, device) -> dict:
    """SURVEY §8 rows f1 / f2 in the bench line: one 1080p GoP (s=3) per stream through
    the proxy codec, then the sender's residual enhancement layer (downscale,
    residual against the decoded working images, sparsify, range encode) and
    the receiver's (range decode, apply) -- the reference session's
    residual path (session.py:173-193, 287-296) -- device-resident, CUDA-event
    timed per stage; bitstreams round-trip exactly."""
    import numpy as np
    import torch
    from paper_2602_03529_b200 import _dev, _lib
    from paper_2602_03529_b200.pipeline import GopCodec
    # one GoP per stream of this GPU (the main workload's 64): the range coder
    # is serial per stream, so its throughput grows with the streams in flight
    G, H, W, s = a.streams, a.height, a.width, 3
    frames = make_inputs(list(range(G)), H, W, device, n_sets=1)[0]
    c = GopCodec(G, H, W, s)
    c.set_gop_ids([0] * G)
    h, w = c.h, c.w
    n = h * w * 3
    f64, i16 = torch.float64, torch.int16
    work = torch.empty((G, 9, h, w, 3), device=device)
    avg = torch.empty((G, n), dtype=f64, device=device)
    dense = torch.empty((G, n), dtype=i16, device=device)
    mags = torch.empty((G, n), dtype=f64, device=device)
    count = torch.empty((G,), dtype=torch.int32, device=device)
    cap = n // 2 + 64
    idx_ws = torch.empty((G * n,), dtype=torch.int64, device=device)
    pay = torch.empty((G * cap,), dtype=torch.uint8, device=device)
    plen = torch.empty((G,), dtype=torch.int64, device=device)
    dec = torch.empty((G, n), dtype=i16, device=device)
    status = torch.empty((G,), dtype=torch.int32, device=device)
    offs = torch.arange(G, dtype=torch.int64, device=device) * cap
    st = _dev.stream()
    theta, step_q = 0.02, 1.0 / 127.0
    stages = [
        # K1 writes the working frames (the residual's `working` GoP) as it
        # box-filters them: no second read of the full-resolution frames
        ("codec", lambda: (c.encode(frames, G, 0, work=work), c.decode(G, 0))),
        ("residual", lambda: _lib.call("sst_residual", work.data_ptr(), c.img[0].data_ptr(), G, h,
                                       w, theta, step_q, avg.data_ptr(), dense.data_ptr(),
                                       mags.data_ptr(), count.data_ptr(), st)),
        ("range_encode", lambda: _lib.call("sst_rc_encode", dense.data_ptr(), G, n,
                                           idx_ws.data_ptr(), pay.data_ptr(), cap,
                                           plen.data_ptr(), st)),
        ("range_decode", lambda: _lib.call("sst_rc_decode", pay.data_ptr(), offs.data_ptr(),
                                           plen.data_ptr(), G, n, dec.data_ptr(),
                                           status.data_ptr(), st)),
        ("apply", lambda: _lib.call("sst_apply_residual", c.img[0].data_ptr(), dec.data_ptr(),
                                    count.data_ptr(), G, h, w, step_q, st)),
    ]
    times = {}
    for it in range(5):
        for name, fn in stages:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            if it >= 2:
                times.setdefault(name, []).append((e0, e1))
    torch.cuda.synchronize()
    ms = {k: float(np.median([x.elapsed_time(y) for x, y in v])) for k, v in times.items()}
    tot = sum(ms.values())
    roundtrip = bool(torch.equal(dec, dense)) and bool((status == 0).all())
    pipe = residual_pipelined(a, device, frames, G, H, W, s, theta, step_q)
    return {"workload": f"{G} x {H}p GoPs, s=3, residual theta={theta}, step 1/127, "
                        "moving-square / noisy-motion synthetic streams",
            "stage_ms": {k: round(v, 3) for k, v in ms.items()},
            "frames_per_s": pipe["frames_per_s"],
            "serial_frames_per_s": round(G * GOP / tot * 1e3, 1),
            "pipelined": pipe,
            "entries_per_gop": round(float(count.float().mean()), 1),
            "payload_bytes_per_gop": round(float(plen.float().mean()), 1),
            "roundtrip_exact": roundtrip and pipe["roundtrip_exact"],
            "range_coder": "encoder: symbols and the adaptive model's per-symbol state computed "
                           "in parallel, one warp per stream codes them (csrc/residual.cu rcp::); "
                           "decoder: one warp per stream (one-warp CTAs, split cumulative "
                           "table, k_rc_decode_x); bytes identical to the reference"}


def residual_pipelined(a, device, frames, G, H, W, s, theta, step_q, depth=6, steps=18) -> dict:
    """The residual workload as a stream of steps: the range decoder is a serial
    chain per stream that occupies one warp of an SM (64 .. 512 streams decode
    in the same time: scripts/rc_decode_micro.py), so the receiver's decode +
    apply of step k, and the sender's range encode (also one warp per
    stream), run on a per-step CUDA stream while the next steps' proxy codec
    and residual kernels run on the main one -- `depth` sets of codec /
    payload / scan buffers rotate (a set is busy for ~20 ms of serial coding),
    and a set is reused only after its previous decode + apply finished.
    Every step's decoded scans are checked against its encoded ones."""
    import numpy as np
    import torch
    from paper_2602_03529_b200 import _dev, _lib
    from paper_2602_03529_b200.pipeline import GopCodec
    main = _dev.stream()
    cur = torch.cuda.current_stream(device)
    h, w = (H + s - 1) // s, (W + s - 1) // s
    n = h * w * 3
    f64, i16 = torch.float64, torch.int16
    cap = n // 2 + 64
    work = torch.empty((G, 9, h, w, 3), device=device)
    avg = torch.empty((G, n), dtype=f64, device=device)
    mags = torch.empty((G, n), dtype=f64, device=device)
    offs = torch.arange(G, dtype=torch.int64, device=device) * cap
    sets = []
    for _ in range(depth):
        c = GopCodec(G, H, W, s)
        c.set_gop_ids([0] * G)
        sets.append(dict(
            c=c, stream=torch.cuda.Stream(device=device),
            dense=torch.empty((G, n), dtype=i16, device=device),
            idx_ws=torch.empty((G * n,), dtype=torch.int64, device=device),
            count=torch.empty((G,), dtype=torch.int32, device=device),
            pay=torch.empty((G * cap,), dtype=torch.uint8, device=device),
            plen=torch.empty((G,), dtype=torch.int64, device=device),
            dec=torch.empty((G, n), dtype=i16, device=device),
            status=torch.empty((G,), dtype=torch.int32, device=device),
            done=None))
    ok = [True]

    def step(k, check):
        S = sets[k % depth]
        c = S["c"]
        if S["done"] is not None:
            cur.wait_event(S["done"])                # set free: its last decode + apply ended
        if check and k >= depth:
            ok[0] &= bool(torch.equal(S["dec"], S["dense"])) and bool((S["status"] == 0).all())
        c.encode(frames, G, 0, work=work)
        c.decode(G, 0)
        _lib.call("sst_residual", work.data_ptr(), c.img[0].data_ptr(), G, h, w, theta, step_q,
                  avg.data_ptr(), S["dense"].data_ptr(), mags.data_ptr(), S["count"].data_ptr(),
                  main)
        sent = torch.cuda.Event()
        sent.record(cur)
        rs = S["stream"]
        rs.wait_event(sent)
        with torch.cuda.stream(rs):
            _lib.call("sst_rc_encode", S["dense"].data_ptr(), G, n, S["idx_ws"].data_ptr(),
                      S["pay"].data_ptr(), cap, S["plen"].data_ptr(), _dev.stream())
            _lib.call("sst_rc_decode", S["pay"].data_ptr(), offs.data_ptr(), S["plen"].data_ptr(),
                      G, n, S["dec"].data_ptr(), S["status"].data_ptr(), _dev.stream())
            _lib.call("sst_apply_residual", c.img[0].data_ptr(), S["dec"].data_ptr(),
                      S["count"].data_ptr(), G, h, w, step_q, _dev.stream())
            S["done"] = torch.cuda.Event()
            S["done"].record(rs)

    for k in range(depth):
        step(k, False)
    for S in sets:
        cur.wait_event(S["done"])
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(cur)
    for S in sets:
        S["stream"].wait_stream(cur)
    for k in range(depth, depth + steps):
        step(k, False)
    for S in sets:
        cur.wait_event(S["done"])
    t1.record(cur)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    for S in sets:
        ok[0] &= bool(torch.equal(S["dec"], S["dense"])) and bool((S["status"] == 0).all())
    return {"depth": depth, "steps": steps, "ms_per_step": round(ms, 3),
            "frames_per_s": round(G * GOP / ms * 1e3, 1), "roundtrip_exact": ok[0],
            "how": "range encode + range decode + apply of step k on a per-step CUDA stream "
                   "(the coders are one warp per stream, serial per stream) while the next "
                   "steps' codec + residual kernels run on the main stream; timed from the "
                   "first step's start to the last step's decode + apply (pipeline drain "
                   "included); per-GoP latency unchanged (~ the serial sum)"}


# ---------------------------------------------------------------------------
# learned tokenizer leg: tcgen05 implicit-GEMM convs

def measured_bf16_peak():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["bf16_tflops"]), "measured burst (MEASURED_PEAKS.json bf16_tflops)"
    except Exception:
        return 2250.0, "nominal dense bf16 (no MEASURED_PEAKS.json)"


def measured_i8_peak(device) -> tuple:
    """The int8 tensor roofline denominator: 2 x MEASURED_PEAKS.json's
    measured bf16 burst (B200's dense int8 rate is twice bf16, like fp8:
    B200_PROFILING.md's table) -- MEASURED_PEAKS.json has no int8 entry.
    Returned with it, as context: the cuBLASLt int8 GEMM measured in this
    run (torch._int_mm, 8192^3, int32 out, best of 10), which reaches a
    smaller fraction of nominal than cuBLAS bf16 does."""
    import torch
    bf, bsrc = measured_bf16_peak()
    lt = None
    try:
        n = 8192
        x = torch.randint(-127, 128, (n, n), dtype=torch.int8, device=device)
        y = torch.randint(-127, 128, (n, n), dtype=torch.int8, device=device)
        for _ in range(3):
            torch._int_mm(x, y)
        best = None
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(x, y)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        del x, y
        lt = round(2 * n ** 3 / (best / 1e3) / 1e12, 1)
    except Exception:                 # pragma: no cover
        pass
    return 2 * bf, f"2 x {bsrc} (B200 dense int8 = 2 x bf16)", lt


def learned_e2e(a, device, model, Codec, s: int) -> dict:
    """The learned codec end to end from pinned HOST frames: each step copies
    the GoPs' frames host -> device, runs the whole codec (encode, FSQ, drop,
    packetise, parse, decode, upscale + blend) and copies the reconstructed
    frames device -> host, inside the timed region; lanes on their own CUDA
    streams overlap the two PCIe directions with compute."""
    import torch
    E, nl, H, W = 8, 4, a.height, a.width
    per = E // nl
    gen = torch.Generator(device=device).manual_seed(1)
    L = []
    for j in range(nl):
        c = Codec(per, H, W, s, model=model)
        c.set_gop_ids(list(range(j * per, (j + 1) * per)))
        h_in = torch.empty((per, GOP, H, W, 3), dtype=torch.float32, pin_memory=True)
        h_in.copy_(torch.rand((per, GOP, H, W, 3), generator=gen, device=device))
        L.append(dict(codec=c, h_in=h_in, h_out=torch.empty_like(h_in, pin_memory=True),
                      d_in=torch.empty((per, GOP, H, W, 3), device=device),
                      d_out=torch.empty((per, GOP, H, W, 3), device=device),
                      stream=torch.cuda.Stream(device=device), k=c.drop_k(a.drop)))

    def one():
        for ln in L:
            with torch.cuda.stream(ln["stream"]):
                ln["d_in"].copy_(ln["h_in"], non_blocking=True)
                ln["codec"].step(ln["d_in"], ln["d_out"], per, drop_k=ln["k"])
                ln["h_out"].copy_(ln["d_out"], non_blocking=True)

    main = torch.cuda.current_stream()
    for _ in range(2):
        one()
    torch.cuda.synchronize()
    K = 5
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for ln in L:
        ln["stream"].wait_stream(main)
    for _ in range(K):
        one()
    for ln in L:
        main.wait_stream(ln["stream"])
    e1.record(main)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    nbytes = E * GOP * H * W * 3 * 4
    return {"value": round(E * GOP / ms * 1e3, 1), "unit": UNIT, "h2d_bytes_per_step": nbytes,
            "d2h_bytes_per_step": nbytes, "gops_per_step": E, "lanes": nl,
            "path": "pinned host frames -> learned codec step -> pinned host frames, per lane "
                    "stream, all inside the timed region"}


def run_learned(a, device, precision: str = "i8") -> dict:
    """G 1080p GoPs per step through the learned codec (encoder + FSQ ->
    similarity -> 10% drop -> packetise -> parse / reassemble -> decoder ->
    upscale + blend), device-resident, CUDA-event timed; plus one serialised
    step timing every tensor-core layer for the roofline.  precision "i8":
    the exact int8 network on tcgen05 kind::i8 (learned_i8.py, the default);
    "bf16": the bf16 network (learned.py)."""
    import numpy as np
    import torch
    G, s, H, W = a.learned_gops, 3, a.height, a.width
    if precision == "i8":
        from paper_2602_03529_b200.learned_i8 import (LearnedI8Config as Cfg,
                                                      LearnedI8GopCodec as Codec)
        from oracle import learned_i8_oracle as LO
    else:
        from paper_2602_03529_b200.learned import LearnedConfig as Cfg, LearnedGopCodec as Codec
    cfg = Cfg()
    codec = Codec(G, H, W, s, cfg=cfg)        # full batch: serialised roofline pass
    model = codec.model
    gen = torch.Generator(device=device).manual_seed(0)
    frames = [torch.rand((G, GOP, H, W, 3), generator=gen, device=device) for _ in range(2)]
    outs = [torch.empty_like(frames[0]) for _ in range(2)]
    drop_k = codec.drop_k(a.drop)
    codec.set_gop_ids(list(range(G)))
    nl = max(1, a.learned_lanes)
    cuts = [G * j // nl for j in range(nl + 1)]
    lanes = []
    for j in range(nl):
        n = cuts[j + 1] - cuts[j]
        c = Codec(n, H, W, s, model=model)
        c.set_gop_ids(list(range(cuts[j], cuts[j + 1])))
        lanes.append(dict(codec=c, sl=slice(cuts[j], cuts[j + 1]), n=n,
                          stream=torch.cuda.Stream(device=device)))

    def step(k):
        codec.step(frames[k % 2], outs[k % 2], G, drop_k=drop_k)

    def lanes_step(k):
        for ln in lanes:
            with torch.cuda.stream(ln["stream"]):
                ln["codec"].step(frames[k % 2][ln["sl"]], outs[k % 2][ln["sl"]], ln["n"],
                                 drop_k=drop_k)

    main = torch.cuda.current_stream()
    for ln in lanes:
        ln["stream"].wait_stream(main)
    for k in range(max(a.warmup, 3)):
        lanes_step(k)
    for ln in lanes:
        main.wait_stream(ln["stream"])
    step(0)
    torch.cuda.synchronize()
    K = max(a.steps // 2, 5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for ln in lanes:
        ln["stream"].wait_stream(main)
    for k in range(K):
        lanes_step(k + 1)
    for ln in lanes:
        main.wait_stream(ln["stream"])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    # one stream alone (G = 1, blend on): GoP latency vs the real-time budget
    c1 = Codec(1, H, W, s, model=model)
    c1.set_gop_ids([0])
    k1 = c1.drop_k(a.drop)
    for k in range(3):
        c1.step(frames[k % 2][:1], outs[k % 2][:1], 1, drop_k=k1)
    torch.cuda.synchronize()
    single = []
    for k in range(10):
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record()
        c1.step(frames[k % 2][:1], outs[k % 2][:1], 1, drop_k=k1)
        b1.record()
        torch.cuda.synchronize()
        single.append(b0.elapsed_time(b1))
    single.sort()
    del c1
    e2e = learned_e2e(a, device, model, Codec, s)
    # serialised pass (full batch, one stream): time every tensor-core layer
    times = []
    orig = model._conv

    def timed(name, x, in_shape, out_grid, taps, t_lo, t_cnt, epi, **kw):
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record()
        orig(name, x, in_shape, out_grid, taps, t_lo, t_cnt, epi, **kw)
        b1.record()
        N, Kd = model.W[name].shape
        nt = taps[0] if isinstance(taps, tuple) else len(taps)
        tok = in_shape[0] * out_grid[0] * out_grid[1]
        if nt == 18:
            # useful work = issued work: t = 1 sees both temporal taps, t = 0
            # only its own (both kernels skip the all-padding t-1 tap there)
            flops = 2 * tok * N * (Kd + Kd // 2)
        else:
            flops = 2 * tok * t_cnt * N * Kd
        times.append((name, nt, b0, b1, flops))

    model._conv = timed
    l0 = model.launches
    try:
        step(1)
        torch.cuda.synchronize()
    finally:
        model._conv = orig
    launches_step = (model.launches - l0) + (1 if drop_k else 0) + 8
    per = [(n, nt, b0.elapsed_time(b1), fl) for n, nt, b0, b1, fl in times]
    halo = [(ms_, fl) for n, nt, ms_, fl in per if nt == 18 and model.W[n].shape[0] % 256 == 0]
    conv_ms = sum(ms_ for _, _, ms_, _ in per)
    if precision == "i8":
        peak, src, cublaslt_i8 = measured_i8_peak(device)
        unit, dtype = "TOP/s", "int8 operands, int32 accumulate (TMEM), exact"
        kern = "k_l8_pair<true> (causal (2,3,3) conv, CTA-pair tcgen05 kind::i8 implicit GEMM)"
    else:
        peak, src = measured_bf16_peak()
        unit, dtype = "TFLOP/s", "bf16 operands, fp32 accumulate (TMEM)"
        kern = "k_lt_convpair<true> (causal (2,3,3) conv, CTA-pair tcgen05 implicit GEMM)"
    achieved = sum(fl for _, fl in halo) / sum(m for m, _ in halo) / 1e9
    res = {
        "precision": precision,
        "lanes": nl,
        "workload": f"{G} x 1080p GoPs per step, s=3, learned causal conv tokenizer "
                    f"(D={cfg.dim}, {cfg.blocks} residual blocks per side, window attention, "
                    f"FSQ 2x(8,8,8,5,5,5)), {int(a.drop * 100)}% intelligent drop, blend n=2; "
                    f"random-init weights",
        "value": round(G * GOP / ms * 1e3, 1), "unit": UNIT, "ms_per_step": round(ms, 3),
        "roofline": {"kernel": kern, "bound": "tensor", "achieved": round(achieved, 1),
                     "peak": round(peak, 1), "unit": unit, "frac": round(achieved / peak, 4),
                     "peak_source": src,
                     "counted": "useful MACs (= issued: the t=0 zero-padding tap is skipped)",
                     "ops_per_launch": halo and int(sum(fl for _, fl in halo) / len(halo)),
                     "avg_launch_ms": round(sum(m for m, _ in halo) / len(halo), 4),
                     "launches_per_step": len(halo)},
        "conv_share_of_serialised_step": round(conv_ms / max(ms, 1e-9), 3),
        "single_stream": {"stream": "1 x 1080p, s=3, learned tokenizer, 10% drop, blend n=2",
                          "gop_ms_median": round(single[len(single) // 2], 3),
                          "gop_ms_max": round(single[-1], 3),
                          "realtime_30fps_budget_ms_per_gop": round(GOP / 30 * 1e3, 1)},
        "gpu_launches_per_step": launches_step,
        "dtype": dtype,
        "e2e": e2e,
    }
    if precision == "i8":
        res["roofline"]["cublaslt_i8_gemm_tops"] = cublaslt_i8
        ops = model.ops_per_gop(codec.Ht, codec.Wt) * G
        res["tensor_tops_path"] = round(ops / ms / 1e9, 1)
        # parity at the bench's own size: one 1080p GoP, GPU vs the exact oracle
        fr0 = frames[0][:1]
        codes, idx, mask, hw = model.encode_frames(fr0, s)
        oc, oi, _ = LO.encode(fr0.cpu().numpy(), s, model.host_weights)
        dec = model.decode_tokens(codes, mask, hw).cpu().numpy()
        od = LO.decode(oc, np.ones(oc.shape[:-1], np.uint8), hw, model.host_weights)
        res["parity_1080p"] = {
            "fsq_index_agreement": float((idx.cpu().numpy() == oi).mean()),
            "decoded_frames_bit_exact": bool(np.array_equal(dec, od)),
            "max_abs_err": float(np.abs(dec - od).max()),
            "oracle": "oracle/learned_i8_oracle.py (exact integer restatement, unpinned: no "
                      "reference model)"}
    else:
        res["tensor_tflops_path"] = round(model.flops_per_gop(codec.Ht, codec.Wt) * G / ms / 1e9, 1)
        res["parity"] = "tests/test_gpu_learned.py vs oracle/learned_oracle.py (torch fp32, unpinned)"
    return res


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(a) -> int:
    """`python bench.py --gpus N` (N > 1) without a torchrun environment:
    re-execute this script under torch.distributed.run with N local ranks
    (one process per GPU, rendezvous on 127.0.0.1) and pass its exit status
    through.  Rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", str(Path(__file__).resolve())] + sys.argv[1:]
    print(f"[bench] launching {a.gpus} ranks: {' '.join(cmd[1:6])} ...", file=sys.stderr,
          flush=True)
    import subprocess
    return subprocess.call(cmd, env=dict(os.environ, OMP_NUM_THREADS="1"))


def comm_info(world: int, dev) -> dict:
    import torch
    import torch.distributed as dist
    info = {"world_size": world, "backend": dist.get_backend() if world > 1 else None,
            "data_path_collectives": 0,
            "collectives": "barrier + max-over-ranks step time + per-rank timing gather"}
    try:
        v = torch.cuda.nccl.version()
        info["nccl_version"] = ".".join(str(x) for x in v) if isinstance(v, tuple) else v
    except Exception:
        pass
    return info


def selftest_launcher(a, rank, world) -> None:
    """CPU path of the N-rank bench (tests/test_bench_cpu.py): gloo rendezvous,
    stream sharding, max-over-ranks of a synthetic per-rank step time, the
    per-rank gather and the JSON line -- everything but the GPU work."""
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    mine = my_streams(a, rank, world)
    ms = 10.0 + rank                                   # rank r "takes" 10 + r ms
    ms_max = max_over_ranks(ms, "cpu") if world > 1 else ms
    per_rank = gather_ranks([ms, len(mine), sum(mine)], "cpu")
    if rank == 0:
        frames = total_streams(a, world) * GOP * a.steps
        line = {"metric": METRIC, "value": round(frames / (ms_max / 1000.0), 2), "unit": UNIT,
                "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "scaling": a.scaling,
                "selftest": True, "ms_max": ms_max, "comm": comm_info(world, "cpu"),
                "per_rank": [{"rank": r, "ms": v[0], "n_streams": int(v[1]),
                              "stream_id_sum": int(v[2])} for r, v in enumerate(per_rank)]}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    a = parse_args()
    in_launch = "WORLD_SIZE" in os.environ
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if a.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if in_launch and world != a.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {a.gpus}: refusing to "
                         f"report a {a.gpus}-GPU number from {world} rank(s)")
    if a.gpus > 1 and not in_launch and a.impl == "ours":
        sys.exit(self_launch(a))
    if a.selftest_launcher:
        return selftest_launcher(a, rank, world)
    base = {"metric": METRIC, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "higher_is_better": True, "scaling": a.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(a)}

    if a.impl == "reference":
        # the reference is a CPU package: rank 0 alone runs it on the host cores
        if rank != 0:
            return
        r = run_reference(a)
        rec = r["record"]
        line = dict(base, impl="reference", value=rec["value"],
                    ms_per_step=round(r["ms"], 2), cpu_baseline=rec,
                    e2e={"value": rec["value"], "unit": UNIT,
                         "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                    psnr_db=round(r["psnr"], 3))
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    # SST_BENCH_SHARE_GPU=1 (test hook): ranks share the visible GPUs round-robin
    # and rendezvous over gloo, so the N>1 control flow (barriers, max-over-ranks,
    # stream sharding) can be exercised on a one-GPU box.  Never used by the driver.
    share = os.environ.get("SST_BENCH_SHARE_GPU") == "1"
    ngpu = torch.cuda.device_count()
    if not share and world > ngpu:
        raise SystemExit(f"bench.py: {world} ranks but only {ngpu} visible GPU(s); "
                         f"one process per GPU is required")
    if share:
        local_rank = local_rank % ngpu
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    res = run_ours(a, rank, world, local_rank)
    if rank == 0:
        line = dict(base, value=round(res["value"], 2), ms_per_step=round(res["ms"] / a.steps, 3),
                    roofline=res["roofline"], gpu_launches=res["launches"],
                    clocks=res["clocks"],
                    stages={k: {"ms_per_launch": round(v[0] / v[1], 4), "launches": v[1]}
                            for k, v in res["stages"].items()},
                    path_roofline=path_roofline(a, res["value"] / world),
                    psnr_db=res["psnr"], per_rank=res["per_rank"],
                    comm=comm_info(world, dev))
        if share and world > 1:
            line["shared_gpu_test_hook"] = True
        line["e2e"] = res.get("e2e")
        if world == 1 and not a.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(a)
            line["parity"] = parity_sample(a, dev)
            line["single_stream"] = single_stream_latency(a, dev)
            line["loss_recovery"] = loss_legs(a, dev)
            line["residual_layer"] = residual_leg(a, dev)
            if a.height == 1080 and a.width == 1920:
                line["small_configs"] = small_configs(a, dev)
        if world == 1 and not a.no_rgb24:
            line["raw_rgb24"] = rgb24_leg(a, rank, world, local_rank, dev)
        if world == 1 and not a.no_learned:
            line["learned_tokenizer"] = run_learned(a, dev, "i8")
            if not a.no_learned_bf16:
                line["learned_tokenizer_bf16"] = run_learned(a, dev, "bf16")
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
