"""Per-step trace of one convoy run (diagnostics): truth / MAP cardinality, parents, kept
hypotheses, pairs, the MAP hypothesis weight, and flags of the reweighted pairs."""
import json
import sys

import numpy as np

sys.path.insert(0, '.')
from paper_2512_06230_b200 import _lib
from paper_2512_06230_b200.build import build

build()
_lib.glmb_init(0)
from paper_2512_06230_b200.scenes import ConvoyConfig, convoy_scene
from paper_2512_06230_b200.tracker import ConvoyTracker

N, H, seed = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
k0, k1 = int(sys.argv[4]), int(sys.argv[5])
cfg = ConvoyConfig(N=N, H_max=H, seed=seed)
Zs, truth, bm, bc = convoy_scene(cfg)
tr = ConvoyTracker(cfg, max(len(z) for z in Zs), K_cap=4096)
tr.reset(bm, bc)
for k in range(k1):
    r = tr.update(k, Zs[k])
    if k < k0:
        continue
    e = tr.estimate(r.T_k)
    kept = r.n_kept
    kw = tr.hu.keep_w[:kept].cpu().numpy()
    fl = tr.pu.flags[:r.n_pairs].cpu().numpy()
    ln = tr.pu.log_norm[:r.n_pairs].cpu().numpy()
    print(json.dumps({"k": k, "M": r.M, "Tk": r.T_k, "truth_n": len(truth[k]), "est_n": len(e), "npar": r.n_parents,
                      "kept": kept, "pairs": r.n_pairs, "kw_top": kw[:3].round(4).tolist(),
                      "flag1": int((fl & 1).sum()), "ln_min": float(ln.min()) if len(ln) else None}))
