#!/usr/bin/env python
"""Hot SASS blocks of one kernel from `ncu -i rep --page source --csv` output (first kernel
section): consecutive instructions with the same execution count are grouped; prints the
top blocks by warp instructions executed with their stall samples and average active
threads.  usage: python profiles/sass_hotspots.py source.csv [top]"""
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
    hdr = rows[starts[0] + 1]
    data = [r for r in rows[starts[0] + 2:starts[1]] if len(r) == len(hdr)]
    ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
    st, at = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Avg. Threads Executed")
    tot = sum(int(r[ie] or 0) for r in data)
    sst = sum(int(r[st] or 0) for r in data)
    print(f"{rows[starts[0]][1]}: {tot} warp instructions, {len(data)} SASS, {sst} stall samples")
    blocks = []
    for i, r in enumerate(data):
        v = int(r[ie] or 0)
        if blocks and blocks[-1][1] == v:
            blocks[-1][2] += 1
            blocks[-1][3] += int(r[st] or 0)
        else:
            blocks.append([i, v, 1, int(r[st] or 0), r[at], r[src].strip()[:60]])
    blocks.sort(key=lambda b: -b[1] * b[2])
    for b in blocks[:top]:
        print(f"sass#{b[0]:5d} count {b[1]:9d} x {b[2]:4d} = {b[1] * b[2] / tot * 100:5.2f}%  "
              f"stalls {b[3] / max(sst, 1) * 100:5.2f}%  thr {b[4]:>5s}  {b[5]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
