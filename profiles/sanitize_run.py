"""Every libglmb kernel once on small inputs (configs 0-1 shapes), written to run under `compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python
profiles/sanitize_run.py` (the tool is closed on this pool; profiles/README.md)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_06230_b200 import _lib as L  # noqa: E402
from paper_2512_06230_b200.build import build  # noqa: E402
from paper_2512_06230_b200 import scenes  # noqa: E402
from paper_2512_06230_b200.step import GlmbStep  # noqa: E402
from paper_2512_06230_b200.hyp import HypothesisUpdate, ParticleUpdate  # noqa: E402

build()
torch.cuda.set_device(0)
L.glmb_init(0)
dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
for cfg_id in (0, 1):
    sc = scenes.make_scene(cfg_id, steps=1)
    st = GlmbStep(sc)
    st.run(0)                                     # predict, birth, compat, reweight
    st.reweight(0, out_of_place=True)             # cluster reweight, out of place
    T, M = st.T_local, len(sc.Z[0])
    C, G = st.out.C_tracks, st.out.gate
    pm, plw, ps = scenes.hypothesis_inputs(T, 0, 3, seed=cfg_id)
    hu = HypothesisUpdate(T, M, 3, 16, 8)
    lc = dv(np.array([-1.0, -0.5, -0.7, -2.0]))
    hu.run(C, G, M, dv(ps), dv(pm.view(np.int32)), dv(plw), sc.cfg.p_d, sc.cfg.kappa, 1e-5, 3, 0, count_lp=lc)
    pu = ParticleUpdate(T, M, 8, st.P)
    pu.run(st.particles, st.Z[0], st.R, hu.keep_idx, 8, hu.alive, hu.theta, M, 3, 0, n_hyp_dev=hu.n_kept)
    est = torch.zeros(T, 3, dtype=torch.float64, device="cuda")
    L.glmb_map_estimate(hu.n_kept, pu.pair_of.view(-1)[:T], pu.out, est)
    mask = torch.zeros(8, hu.ldt, dtype=torch.int32, device="cuda")
    L.glmb_next_parents(hu.n_kept, hu.keep_w, pu.pair_of.view(-1)[:8 * T].view(8, T), T, 1, T - 1, mask,
                        torch.zeros(8, dtype=torch.float64, device="cuda"),
                        torch.zeros(1, dtype=torch.int32, device="cuda"))
    bufs = [torch.zeros_like(C), torch.zeros_like(G)]
    L.glmb_compat_peers(st.particles, st.Z[0], st.R, sc.cfg.p_d, sc.cfg.kappa, sc.cfg.gamma, None,
                        torch.tensor([bufs[0].data_ptr()], dtype=torch.int64, device="cuda"),
                        torch.tensor([bufs[1].data_ptr()], dtype=torch.int64, device="cuda"), 0,
                        C.shape[1], G.shape[1])
    torch.cuda.synchronize()
    print(f"cfg{cfg_id}: all kernels ran")
