#!/usr/bin/env python
"""compat at cfg3's tracks and clouds for several measurement counts M (diagnostic): the scene's
Z_k truncated or padded with copies, mean launch time over `reps`, pairs/clk/SM at 1965 MHz --
how much of the cfg3 rate is lost to the ragged last measurement tile and the grid's tail."""
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
sc = make_scene(3, steps=1)
st = GlmbStep(sc)
for k in range(25):
    st.predict(k)
st.birth(0)
Z0 = sc.Z[0]
reps = 10
for M in [int(m) for m in (sys.argv[1:] or ["1024", "1198", "1280", "2048", "2560", "4701"])]:
    Z = np.resize(Z0, (M, 2)).astype(np.float32)
    Zd = torch.from_numpy(Z).cuda()
    ldc = (M + 31) // 32 * 32
    C = torch.zeros(st.T_local, ldc, device="cuda")
    G = torch.zeros(st.T_local, ldc // 32, dtype=torch.int32, device="cuda")
    c = sc.cfg
    for _ in range(2):
        L.glmb_compat(st.particles, Zd, c.R, c.p_d, c.kappa, c.gamma, None, C, G)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        L.glmb_compat(st.particles, Zd, c.R, c.p_d, c.kappa, c.gamma, None, C, G)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    pairs = M * st.T_local * st.P
    print(f"M {M:5d}  {ms:7.3f} ms  {pairs / ms * 1e3 / (148 * 1.965e9):6.2f} pairs/clk/SM", flush=True)
