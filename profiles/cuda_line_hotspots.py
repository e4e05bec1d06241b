#!/usr/bin/env python
"""Per CUDA source line: warp instructions executed and stall samples, from
`ncu -i rep --page source --csv --print-source cuda,sass`, for every kernel in the report
(or only those whose name contains FILTER).
usage: python profiles/cuda_line_hotspots.py report.ncu-rep [top] [FILTER]"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, top=30, flt=""):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    per_fn = collections.OrderedDict()
    fname, fn, hdr = None, None, None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            fn = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if fn is None or hdr is None or len(r) != len(hdr) or flt not in fn:
            continue
        try:
            line = int(r[0])
        except ValueError:
            continue
        d = per_fn.setdefault(fn, (collections.Counter(), collections.Counter(), {}))
        key = (fname, line)
        d[2][key] = r[1].strip()[:70]
        d[0][key] += int(r[hdr.index("Instructions Executed")] or 0)
        d[1][key] += int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    for fn, (inst, stall, text) in per_fn.items():
        ti, ts = sum(inst.values()), sum(stall.values())
        print(f"{fn}: {ti} warp instructions, {ts} stall samples")
        for key, v in inst.most_common(top):
            print(f"  {key[0]}:{key[1]:5d} inst {v / max(ti, 1) * 100:5.1f}%  stall "
                  f"{stall[key] / max(ts, 1) * 100:5.1f}%  {text[key]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30, sys.argv[3] if len(sys.argv) > 3 else "")
