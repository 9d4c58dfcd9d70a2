"""Summarise ncu captures (gpurun_out/*.ncu-rep, launches.csv) into profiles/.

    python scripts/ncu_summary.py <tag> <gops_per_captured_launch> <launches.csv> <rep>...

Writes profiles/<tag>_ncu_summary.md (launch list shares + per-kernel key
metrics + top stall reasons) and profiles/<tag>_traffic.json (DRAM bytes per
launch per kernel, consumed by bench.py's roofline.traffic).
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import Counter, defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
NCU = "/usr/local/cuda/bin/ncu"
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]
KERNEL_KEY = {"k_encode": "K1_encode", "k_upscale_blend": "K5_upscale_blend",
              "k_decode": "K4_unpack_decode", "k_packetize": "K3_packetize",
              "k_topk": "K2_select_drop", "k_parse": "K4_parse"}


def _raw(rep: Path):
    out = subprocess.run([NCU, "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def _stalls(rep: Path):
    out = subprocess.run([NCU, "-i", str(rep), "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h = rows[1]
    reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
    tot = Counter()
    for r in rows[2:]:
        for x in reasons:
            v = r[h.index(x)]
            tot[x] += int(v) if v.isdigit() else 0
    s = sum(tot.values()) or 1
    return [(k, round(100 * v / s, 1)) for k, v in tot.most_common(5)]


def launches(path: Path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot, cnt = defaultdict(float), Counter()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].replace("void ", "").replace("sst::", "")
        if not name.startswith("k_"):
            continue                                   # input generation etc.
        short = name.split("(")[0]
        tot[short] += float(r[vi].replace(",", ""))
        cnt[short] += 1
    return tot, cnt


def main():
    tag, gops = sys.argv[1], int(sys.argv[2])
    lcsv, reps = Path(sys.argv[3]), [Path(p) for p in sys.argv[4:]]
    md = [f"# ncu summary — {tag}", ""]
    tot, cnt = launches(lcsv)
    T = sum(tot.values())
    md += ["## Launch list (our kernels only; `ncu --metrics gpu__time_duration.sum "
           "--clock-control none -k regex:^k_` over `python bench.py --steps 2 --warmup 1 "
           "--no-e2e --no-cpu-baseline`, i.e. the bench workload: 64 x 1080p streams, 32 GoPs "
           "per launch; cold-cache and serialised, so compare shares)", "",
           "| kernel | launches | total µs | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        md.append(f"| `{k}` | {cnt[k]} | {v / 1000:.1f} | {100 * v / T:.1f}% |")
    traffic = {"_source": f"profiles/{tag}_ncu_summary.md (ncu --set full)",
               "_unit": "DRAM bytes (read + write) per GoP; bench.py multiplies by GoPs per launch"}
    for rep in reps:
        h, units, data = _raw(rep)
        if not data:
            continue
        r = data[0]
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else rep.stem
        md += ["", f"## `{name.split('(')[0]}` ({rep.name})", "", "| metric | value |", "|---|---|"]
        vals = {}
        for key, label in METRICS:
            if key in h:
                vals[key] = r[h.index(key)]
                md.append(f"| {label} (`{key}`) | {r[h.index(key)]} {units[h.index(key)]} |")
        st = _stalls(rep)
        if st:
            md.append(f"| top stall reasons | {', '.join(f'{k} {v}%' for k, v in st)} |")
        try:
            def tobytes(key):
                v = float(vals[key].replace(",", ""))
                u = units[h.index(key)].lower()
                return v * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)
            dram = tobytes("dram__bytes_read.sum") + tobytes("dram__bytes_write.sum")
            for k, v in KERNEL_KEY.items():
                if k in name:
                    traffic[v] = int(dram / gops)
        except Exception:
            pass
    out = ROOT / "profiles" / f"{tag}_ncu_summary.md"
    out.write_text("\n".join(md) + "\n")
    (ROOT / "profiles" / f"{tag}_traffic.json").write_text(json.dumps(traffic, indent=1))
    print(out)


if __name__ == "__main__":
    main()
