#!/usr/bin/env python
"""DRAM traffic per launch of each kernel class from one `ncu --set full`
capture of a bench workload (dram__bytes_read.sum + dram__bytes_write.sum),
written to profiles/ncu_traffic_<tag>.json tagged with the library build id,
so bench.py reports `roofline.traffic` only from a capture of the build it
runs. Multi-kernel classes (K1 Q-step + col_reduce) are summed per step.

  traffic_from_ncu.py REPORT.ncu-rep WORKLOAD TAG
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2306_08881_b200"))


def kclass(name):
    n = name.replace(" ", "")
    if "orth_kernel" in n:
        return "orth"
    if "col_reduce" in n:
        return "proj_q"
    m = re.search(r"stream_kernel<\(int\)(\d)", n) or re.search(r"stream_kernel<(\d)", n)
    if m:
        return {"0": "proj_p", "3": "proj_q", "2": "decode_q"}[m.group(1)]
    m = re.search(r"row_kernel<\(int\)(\d)", n) or re.search(r"row_kernel<(\d)", n)
    if m:
        return {"0": "proj_p", "1": "decode_p", "2": "decode_q", "3": "decode_q"}[m.group(1)]
    if "tc5_k1p" in n or "k1p_kernel" in n:
        return "proj_p"
    m = re.search(r"tc5_decode_kernel<\(int\)(\d)", n) or re.search(r"tc5_decode_kernel<(\d)", n)
    if m:
        return {"2": "decode_p", "3": "decode_q"}[m.group(1)]
    m = re.search(r"tc_kernel<\(int\)(\d)", n) or re.search(r"tc_kernel<(\d)", n)
    if m:
        return {"0": "proj_p", "1": "proj_q", "2": "decode_p", "3": "decode_q"}[m.group(1)]
    return None


def main(rep, workload, tag):
    from build import build_id
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    iname, ir, iw = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    units = rows[1]
    scale = lambda u: {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    per = defaultdict(list)
    for r in rows[2:]:
        c = kclass(r[iname])
        if c is None:
            continue
        b = float(r[ir].replace(",", "")) * scale(units[ir]) + float(r[iw].replace(",", "")) * scale(units[iw])
        per[c].append(b)
    # col_reduce follows each K1 Q-step launch: pair them up (one step = both)
    out = {}
    for c, v in per.items():
        if c == "proj_q":
            k1 = [x for x, r in zip(v, [rr for rr in rows[2:] if kclass(rr[iname]) == "proj_q"])
                  if "col_reduce" not in r[iname]]
            red = [x for x, r in zip(v, [rr for rr in rows[2:] if kclass(rr[iname]) == "proj_q"])
                   if "col_reduce" in r[iname]]
            steps = max(1, len(k1))
            out[c] = int((sum(k1) + sum(red)) / steps)
        else:
            out[c] = int(sum(v) / len(v))
    path = os.path.join(ROOT, "profiles", f"ncu_traffic_{tag}.json")
    data = {}
    if os.path.exists(path):
        data = json.load(open(path))
    data["build_id"] = build_id()
    data["_source"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per launch (per step for proj_q: K1 "
                       f"+ col_reduce) from `ncu --set full` captures of bench.py on 1x B200, build {build_id()}")
    data[workload] = out
    json.dump(data, open(path, "w"), indent=1)
    print(path, workload, out)


if __name__ == "__main__":
    main(*sys.argv[1:4])
