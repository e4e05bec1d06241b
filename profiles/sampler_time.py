#!/usr/bin/env python
"""Standalone timing of glmb_assoc_sample on cfg3's C_k (diagnostic): H_old = 100 parents x
H_up = 100 samples, R launches back to back between two events behind a busy GPU, mean us per
launch; also the whole HypothesisUpdate chain."""
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
args = (st.out.C_tracks, st.out.gate, M, dv(ps), dv(pm.view(np.int32)), dv(plw), c.p_d, c.kappa, 1e-5, c.seed, 0)
for _ in range(3):
    hu.run(*args)
torch.cuda.synchronize()
n = 100 * 100


def sample():
    L.glmb_assoc_sample(100, dv_pm, dv_plw, hu.d[:T], dv_ps, c.p_d, c.kappa, hu.row_ptr, hu.col, hu.val, hu.ln_val,
                        M, c.seed, 0, hu.alive[:n], hu.theta[:n], hu.logw[:n], hu.hash[:n], None)


dv_pm, dv_plw, dv_ps = dv(pm.view(np.int32)), dv(plw), dv(ps)
for name, fn in (("assoc_sample", sample), ("hypothesis chain", lambda: hu.run(*args))):
    for R in (1, 10):
        ts = []
        for _ in range(8):
            torch.cuda._sleep(1_000_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(R):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / R)
        ts.sort()
        print(f"{name:17s} x{R:2d}  {sum(ts[1:-1]) / len(ts[1:-1]):7.1f} us")
