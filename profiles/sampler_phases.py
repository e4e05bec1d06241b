#!/usr/bin/env python
"""Phase timeline of assoc_sample at cfg3 (diagnostic; needs a GLMB_SAMP_DEBUG=3 build, whose
kernel stores %globaltimer stamps per CTA -- start, setup done, stage 1 done, stage 2 done,
end -- into the fingerprint output).  Prints the mean phase durations and the spread of CTA
start and end times."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_06230_b200 import _lib as L  # noqa: E402
from paper_2512_06230_b200.hyp import HypothesisUpdate  # noqa: E402
from paper_2512_06230_b200.scenes import hypothesis_inputs, make_scene  # noqa: E402
from paper_2512_06230_b200.step import GlmbStep  # noqa: E402

torch.cuda.set_device(0)
L.glmb_init(0)
sc = make_scene(3, steps=1)
st = GlmbStep(sc)
for k in range(6):
    st.predict(k)
st.birth(0)
st.compat(0)
c = sc.cfg
T, M = st.T_local, len(sc.Z[0])
pm, plw, ps = hypothesis_inputs(c.T, c.B, 100, seed=c.seed)
dv = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
hu = HypothesisUpdate(T, st.M_max, 100, 100, 100)
for _ in range(3):
    hu.run(st.out.C_tracks, st.out.gate, M, dv(ps), dv(pm.view(np.int32)), dv(plw), c.p_d, c.kappa, 1e-5, c.seed, 0)
torch.cuda.synchronize()
raw = hu.hash[:400 * 16].cpu().numpy().astype(np.int64).reshape(400, 16)
order = [0, 10, 11, 12, 13, 14, 1, 2, 3, 4]
names = ["init+zero smem", "filter ballot", "scan", "rows fill", "pw/nzq scans", "theta zero-fill",
         "stage1", "stage2", "finalize"]
ts = raw[:, order]
t0 = ts[:, 0].min()
ts = (ts - t0) / 1e3
d = np.diff(ts, axis=1)
print("CTA start  min/median/max us:", ts[:, 0].min(), np.median(ts[:, 0]), ts[:, 0].max())
print("CTA end    min/median/max us:", ts[:, -1].min(), np.median(ts[:, -1]), ts[:, -1].max())
for name, col in zip(names, d.T):
    print(f"{name:16s} mean {col.mean():7.2f} us  median {np.median(col):7.2f}  max {col.max():7.2f}")
