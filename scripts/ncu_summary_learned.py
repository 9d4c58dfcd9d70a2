"""Summarise the learned-tokenizer ncu captures into profiles/<tag>_learned_ncu_summary.md.

    python scripts/ncu_summary_learned.py <tag> <launches.csv> <rep>...
"""
import csv, io, subprocess, sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
NCU = "/usr/local/cuda/bin/ncu"
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % (active)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe % (elapsed)"),
    ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
     "UTCHMMA bf16->fp32 % of peak (elapsed)"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
]


def raw(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def launches(path):
    agg = defaultdict(lambda: [0.0, 0])
    hdr = None
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"ms": 1000.0, "ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1000.0,
              "nsecond": 1e-3}.get(d["Metric Unit"], 1.0)
        k = d["Kernel Name"].split("(")[0]
        agg[k][0] += v
        agg[k][1] += 1
    return agg


def main():
    tag, lcsv, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    lines = [f"# ncu summary -- learned tokenizer path ({tag})", ""]
    agg = launches(lcsv)
    tot = sum(v[0] for v in agg.values())
    lines += ["## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_` "
              "over `python scripts/learned_step.py 32 2 [i8|bf16]`: 2 steps of the learned codec, 32 x 1080p GoPs, s=3; "
              "cold-cache and serialised, so compare shares)", "",
              "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (v, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
        lines.append(f"| `{k}` | {n} | {v:.1f} | {100 * v / tot:.1f}% |")
    for rep in reps:
        rows, units = raw(rep)
        for d in rows:
            lines += ["", f"## `{d['Kernel Name'][:90]}` ({Path(rep).name})", "", "| metric | value |", "|---|---|"]
            for key, label in METRICS:
                if key in d:
                    lines.append(f"| {label} (`{key}`) | {d[key]} {units.get(key, '')} |")
            # int8 tensor-op paths (kind::i8: UTCIMMA), whatever their exact metric names
            for key in sorted(k for k in d if "utcimma" in k and k.endswith("pct_of_peak_sustained_elapsed")
                              and d[k] not in ("", "0")):
                lines.append(f"| int8 tensor op % of peak (`{key}`) | {d[key]} |")
            stalls = {k: float(v) for k, v in d.items()
                      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                      and v.replace('.', '', 1).isdigit()}
            s = sum(stalls.values()) or 1.0
            top = sorted(stalls.items(), key=lambda x: -x[1])[:5]
            lines.append("| top stall reasons | " + ", ".join(
                f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / s:.1f}%" for k, v in top) + " |")
    out = ROOT / "profiles" / f"{tag}_learned_ncu_summary.md"
    out.write_text("\n".join(lines) + "\n")
    print(out)


if __name__ == "__main__":
    main()
