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
ts = hu.hash[:400 * 6].cpu().numpy().astype(np.int64).reshape(400, 6)[:, :5]
t0 = ts[:, 0].min()
ts = (ts - t0) / 1e3
d = np.diff(ts, axis=1)
print("CTA start  min/median/max us:", ts[:, 0].min(), np.median(ts[:, 0]), ts[:, 0].max())
print("CTA end    min/median/max us:", ts[:, 4].min(), np.median(ts[:, 4]), ts[:, 4].max())
for name, col in zip(("setup", "stage1", "stage2", "finalize"), d.T):
    print(f"{name:9s} mean {col.mean():7.2f} us  median {np.median(col):7.2f}  max {col.max():7.2f}")
