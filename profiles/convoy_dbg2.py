import sys, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2512_06230_b200 import _lib
from paper_2512_06230_b200.build import build
build(); _lib.glmb_init(0)
from paper_2512_06230_b200.scenes import ConvoyConfig, convoy_scene
from paper_2512_06230_b200.tracker import ConvoyTracker
N = int(sys.argv[1]); steps = int(sys.argv[2])
cfg = ConvoyConfig(N=N, H_max=20, K=steps, P=512)
Zs, truth, bm, bc = convoy_scene(cfg)
tr = ConvoyTracker(cfg, max(len(z) for z in Zs), K_cap=256)
tr.reset(bm, bc)
for k in range(steps):
    r = tr.update(k, Zs[k])
    e = tr.estimate(r.T_k)
    hu = tr.hu
    kept = hu.n_kept.item()
    ki = hu.keep_idx[:kept].cpu().numpy()
    al = hu.alive.cpu().numpy()[ki, 0]
    kw = hu.keep_w[:kept].cpu().numpy()
    th = hu.theta.cpu().numpy()[ki[0], :r.M]
    print(k, "Tk", r.T_k, "kept", kept, "pairs", r.n_pairs, "card", len(e), "/", len(truth[k]),
          "w0 %.3f" % kw[0], "nalive", [bin(a).count('1') for a in al[:6]], "theta0", th.tolist()[:15],
          "est", np.round(e, 1).tolist(), "truth", np.round(truth[k], 1).tolist())
