#!/usr/bin/env python
"""Phase timeline of the reweight e-cache kernel at cfg3 (diagnostic; needs a GLMB_RW_DEBUG=3
build, whose kernel stores %globaltimer stamps per unit -- start, S_j collected, fp32 pass 1
done, merge done, pass 2 done -- and the SM id over the unit's first output weights).  Prints
the mean phase durations, the spread of unit start/end times and the units per SM."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_06230_b200 import _lib as L  # noqa: E402
from paper_2512_06230_b200.scenes import make_scene  # noqa: E402
from paper_2512_06230_b200.step import GlmbStep  # noqa: E402

torch.cuda.set_device(0)
L.glmb_init(0)
# argv[1] = N: the state after N steps of predict + reweight (the bench's late-step state), else fresh
N = int(sys.argv[1]) if len(sys.argv) > 1 else 0
sc = make_scene(3, steps=max(N, 1) + 1)
st = GlmbStep(sc)
if N == 0:
    for k in range(6):
        st.predict(k)
else:
    for k in range(N):
        st.predict(k)
        st.birth(k)
        st.reweight(k, out_of_place=True)
K = N
st.birth(K)
for rep in range(4):
    st.reweight(K, out_of_place=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
st.reweight(K, out_of_place=True)
e1.record()
torch.cuda.synchronize()
print(f"launch {e0.elapsed_time(e1) * 1e3:.1f} us (stamped build)")
w = st.weights()
T = st.T_local
ts = w[:, :14].contiguous().view(torch.int64).cpu().numpy()[:, :7]
ok = (np.abs(ts[:, 0] - np.median(ts[:, 0])) < 10**7) & (np.abs(ts[:, 4] - np.median(ts[:, 0])) < 10**7)
print(f"units with stamps: {ok.sum()} of {len(ok)} (the rest took the |S_j| = 0 path)")
ts = ts[ok]
print(f"units rerun in fp64: {int(ts[:, 6].sum())} of {len(ts)}")
sm = ts[:, 5]
ts = ts[:, :5]
t0 = ts[:, 0].min()
ts = (ts - t0) / 1e3
d = np.diff(ts, axis=1)
pc = (0, 10, 50, 90, 99, 100)
print("unit start percentiles", pc, np.round(np.percentile(ts[:, 0], pc), 2))
print("unit end   percentiles", pc, np.round(np.percentile(ts[:, 4], pc), 2))
for name, col in zip(("collect S", "pass 1", "merge", "pass 2"), d.T):
    print(f"{name:10s} mean {col.mean():7.2f} us  median {np.median(col):7.2f}  max {col.max():7.2f}")
tot = ts[:, 4] - ts[:, 0]
print(f"unit total mean {tot.mean():.2f} us")
cnt = np.bincount(sm, minlength=148)
print("units per SM: min", cnt.min(), "max", cnt.max())
# first wave vs second wave
order = np.argsort(ts[:, 0])
first = order[:592]
print(f"first 592 units: total mean {tot[first].mean():.2f}, pass1 mean {d[first, 1].mean():.2f}")
rest = order[592:]
if len(rest):
    print(f"later units: total mean {tot[rest].mean():.2f}, pass1 mean {d[rest, 1].mean():.2f}")
