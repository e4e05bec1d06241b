import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2512_06230_b200 import _lib
from paper_2512_06230_b200.build import build
build(); _lib.glmb_init(0)
from paper_2512_06230_b200.scenes import ConvoyConfig, convoy_scene, ground_track
from paper_2512_06230_b200.tracker import ConvoyTracker
N = int(sys.argv[1]); steps = int(sys.argv[2]); kw = dict(a.split("=") for a in sys.argv[3:])
kw = {k: (float(v) if "." in v else int(v)) for k, v in kw.items()}
cfg = ConvoyConfig(N=N, K=steps, **kw)
Zs, truth, bm, bc = convoy_scene(cfg)
g = ground_track(cfg)
tr = ConvoyTracker(cfg, max(len(z) for z in Zs), K_cap=2048)
tr.reset(bm, bc)
bad = 0
for k in range(steps):
    r = tr.update(k, Zs[k])
    e = tr.estimate(r.T_k)
    if len(e) != len(truth[k]):
        bad += 1
        if bad <= 12:
            print(k, "card", len(e), "/", len(truth[k]), "pairs", r.n_pairs, "kept", r.n_kept, "speed %.2f turn %.3f" % (g[k, 2], (g[min(k+1, steps-1), 3] - g[k, 3]) / cfg.dt),
                  "est", np.round(e, 1).tolist()[:6], "truth", np.round(truth[k], 1).tolist()[:6])
print("bad steps", bad, "of", steps)
