#!/usr/bin/env python
"""Standalone timing of glmb_reweight at cfg3 (diagnostic): back-to-back launches (L2 warm with
the previous launch's tail) and launches after an L2 flush, mean us and fraction of the
measured HBM peak at 16 B per particle."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2512_06230_b200 import _lib as L  # noqa: E402
from paper_2512_06230_b200.scenes import make_scene  # noqa: E402
from paper_2512_06230_b200.step import GlmbStep  # noqa: E402

torch.cuda.set_device(0)
L.glmb_init(0)
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
hbm = float(peak["hbm_gbs"])
sc = make_scene(3, steps=1)
st = GlmbStep(sc)
for k in range(6):
    st.predict(k)
st.birth(0)
nbytes = st.T_local * st.P * 16
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    st.reweight(0, out_of_place=True)
torch.cuda.synchronize()
for mode in ("back-to-back", "after L2 flush"):
    ts = []
    for _ in range(20):
        if mode != "back-to-back":
            flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st.reweight(0, out_of_place=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    us = sum(ts[2:-2]) / len(ts[2:-2])
    print(f"reweight {mode:15s} {us:6.1f} us  {nbytes / us / 1e3:7.1f} GB/s  frac {nbytes / us / 1e3 / hbm:.3f}")
# queued behind a busy GPU: R launches back to back between two events (no host gaps)
for R in (1, 10):
    ts = []
    for _ in range(10):
        flush.fill_(1)
        torch.cuda._sleep(2_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(R):
            st.reweight(0, out_of_place=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / R)
    ts.sort()
    us = sum(ts[2:-2]) / len(ts[2:-2])
    print(f"reweight queued x{R:2d}    {us:6.1f} us  {nbytes / us / 1e3:7.1f} GB/s  frac {nbytes / us / 1e3 / hbm:.3f}")
# the same bytes through a plain elementwise kernel (torch.addcmul: reads x, y, w, writes w_out)
d = st.particles.data
x, y, w = d[0], d[1], st.weights()
wo = torch.empty_like(w)
for R in (1, 10):
    ts = []
    for _ in range(10):
        flush.fill_(1)
        torch.cuda._sleep(2_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(R):
            torch.addcmul(w, x, y, value=0.0, out=wo)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / R)
    ts.sort()
    us = sum(ts[2:-2]) / len(ts[2:-2])
    print(f"addcmul  queued x{R:2d}    {us:6.1f} us  {nbytes / us / 1e3:7.1f} GB/s  frac {nbytes / us / 1e3 / hbm:.3f}")
# theta mode through the pair path: S_j lists built on the host from theta (identity pair_track)
import numpy as np  # noqa: E402
th = sc.theta[0]
T = st.T_local
lists = [[] for _ in range(T)]
for i, t in enumerate(th):
    if t > 0:
        lists[t - 1].append(i)
ptr = np.zeros(T + 1, np.int32)
ptr[1:] = np.cumsum([len(x) for x in lists])
meas = np.array([i for x in lists for i in x] or [0], np.int32)
dv = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
pt, pp, pm_, npairs = dv(np.arange(T, dtype=np.int32)), dv(ptr), dv(meas), dv(np.array([T], np.int32))
wo2 = torch.empty_like(w)
ln2, fl2, ess2 = (torch.empty(T, device="cuda"), torch.empty(T, dtype=torch.int32, device="cuda"),
                  torch.empty(T, device="cuda"))
for R in (1, 10):
    ts = []
    for _ in range(10):
        flush.fill_(1)
        torch.cuda._sleep(2_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(R):
            L.glmb_reweight_pairs(st.particles, st.Z[0], st.R, T, npairs, pt, pp, pm_, wo2, ln2, fl2, ess2)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / R)
    ts.sort()
    us = sum(ts[2:-2]) / len(ts[2:-2])
    print(f"pairs    queued x{R:2d}    {us:6.1f} us  {nbytes / us / 1e3:7.1f} GB/s  frac {nbytes / us / 1e3 / hbm:.3f}")
