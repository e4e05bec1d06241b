#!/usr/bin/env python
"""glmb_reweight at cfg3 after N steps of predict + birth + reweight (diagnostic: the bench's
late-step state vs a fresh one): 10 launches back to back into a scratch buffer, with the
state's own weights and with the weights reset to uniform."""
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
N = int(sys.argv[1]) if len(sys.argv) > 1 else 23
sc = make_scene(3, steps=N + 1)
st = GlmbStep(sc)
for k in range(N):
    st.predict(k)
    st.birth(k)
    st.reweight(k, out_of_place=True)
st.predict(N)
st.birth(N)
torch.cuda.synchronize()
w_out = torch.empty_like(st.weights())
ln, fl = torch.empty_like(st.out.log_norm), torch.empty_like(st.out.flags)


def b2b(reps=10, trials=5):
    out = []
    for _ in range(trials):
        torch.cuda._sleep(1_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            L.glmb_reweight(st.particles, st.Z[N], st.R, st.theta[N], st.col_offset, ln, fl, None, w_out=w_out)
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) * 1e3 / reps)
    return float(np.median(out))


w = st.weights()
wc = w.cpu().numpy()
print(f"N={N}: weights zero {np.mean(wc == 0):.3f}, denormal {np.mean((wc > 0) & (wc < 1.18e-38)):.3f}, "
      f"max per track median {np.median(wc.max(axis=1)):.3g}")
print(f"state weights   {b2b():6.1f} us")
w.fill_(1.0 / st.P)
print(f"uniform weights {b2b():6.1f} us")
