#!/usr/bin/env python
"""Summarise ncu outputs into profiles/ (committed evidence).

  summarize_ncu.py launches <launches.csv> <out.md>    per-kernel share of the launch list
  summarize_ncu.py full <report.ncu-rep> <out.md>      key metrics of a --set full capture
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_sb"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def short(name):
    name = name.replace("void ", "").replace("(anonymous namespace)::", "").replace("acp::", "")
    return name.split("(")[0][:48]


def launches(path, out):
    txt = open(path).read()
    start = txt.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        k = short(r["Kernel Name"])
        tot[k] += v * scale
        cnt[k] += 1
    ours = {k: v for k, v in tot.items() if any(s in k for s in ("row_kernel", "col_kernel", "orth_kernel", "stream_", "k1p_kernel", "fill_kernel", "tc_kernel", "tc5_", "col_reduce", "finite_scan", "nvls", "materialize", "transpose"))}
    all_t = sum(tot.values())
    our_t = sum(ours.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list summary: {path}\n\n")
        f.write("Cold-cache, serialised per-launch times (`--metrics gpu__time_duration.sum "
                "--clock-control none`); compare SHARES, not absolutes.\n\n")
        f.write("| kernel | launches | total us | share of our kernels |\n|---|---|---|---|\n")
        for k, v in sorted(ours.items(), key=lambda x: -x[1]):
            f.write(f"| {k} | {cnt[k]} | {v:.1f} | {100 * v / our_t:.1f}% |\n")
        f.write(f"\nour kernels: {our_t:.1f} us of {all_t:.1f} us total GPU time in the capture "
                f"(the rest is input generation by torch).\n")
    print(open(out).read())


def full(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    units = rows[1]
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary: {path}\n\n")
        cols = [(h.index(k), lab) for k, lab in KEYS if k in h]
        f.write("| kernel | " + " | ".join(f"{lab} ({units[i]})" for i, lab in cols) + " |\n")
        f.write("|---|" + "---|" * len(cols) + "\n")
        for r in rows[2:]:
            f.write(f"| {short(r[h.index('Kernel Name')])} | " + " | ".join(r[i] for i, _ in cols) + " |\n")
    print(open(out).read())


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
