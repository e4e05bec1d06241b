#!/usr/bin/env python
"""Per CUDA source line: warp instructions executed and stall samples, from
`ncu -i rep --page source --csv --print-source cuda,sass` (first kernel in the report).
usage: python profiles/cuda_line_hotspots.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    inst, stall, text = collections.Counter(), collections.Counter(), {}
    fname, fn, hdr, seen_fn = None, None, None, None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            fn = r[1]
            seen_fn = seen_fn or fn
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if fn != seen_fn or hdr is None or len(r) != len(hdr):
            continue
        try:
            line = int(r[0])
        except ValueError:
            continue
        key = (fname, line)
        text[key] = r[1].strip()[:70]
        inst[key] += int(r[hdr.index("Instructions Executed")] or 0)
        stall[key] += int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    ti, ts = sum(inst.values()), sum(stall.values())
    print(f"{seen_fn}: {ti} warp instructions, {ts} stall samples")
    for key, v in inst.most_common(top):
        print(f"{key[0]}:{key[1]:5d} inst {v / ti * 100:5.1f}%  stall {stall[key] / max(ts, 1) * 100:5.1f}%  {text[key]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
