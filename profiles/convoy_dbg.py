import sys, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2512_06230_b200 import _lib
from paper_2512_06230_b200.build import build
build(); _lib.glmb_init(0)
from paper_2512_06230_b200.scenes import ConvoyConfig, convoy_scene
from paper_2512_06230_b200.tracker import ConvoyTracker
cfg = ConvoyConfig(N=int(sys.argv[1]) if len(sys.argv) > 1 else 1, H_max=10, K=40, P=512)
Zs, truth, bm, bc = convoy_scene(cfg)
tr = ConvoyTracker(cfg, max(len(z) for z in Zs), K_cap=128)
tr.reset(bm, bc)
print("birth mean", bm, "truth0", truth[0], "Z0", Zs[0])
for k in range(int(sys.argv[2]) if len(sys.argv) > 2 else 12):
    r = tr.update(k, Zs[k])
    e = tr.estimate(r.T_k)
    hu, pu = tr.hu, tr.pu
    Tk = r.T_k
    d = hu.d[:Tk].cpu().numpy()
    kept = hu.n_kept.item()
    kw = hu.keep_w[:kept].cpu().numpy()
    C = tr.C_tracks[:Tk, :r.M].cpu().numpy()
    ki = hu.keep_idx[:kept].cpu().numpy()
    al = hu.alive.cpu().numpy()[ki, 0]
    th = hu.theta.cpu().numpy()[ki, :r.M]
    lw = hu.logw.cpu().numpy()[ki]
    src = tr.bufs[1 - tr.cur]  # after update cur flipped: src of this step is bufs[1-cur]
    x = src.data[0, :Tk].cpu().numpy(); y = src.data[1, :Tk].cpu().numpy(); w = src.data[5, :Tk].cpu().numpy()
    print(json.dumps({"k": k, "M": r.M, "Tk": Tk, "npar": r.n_parents, "kept": kept, "pairs": r.n_pairs,
        "d": d.round(3).tolist(), "Cmax": C.max(1).round(3).tolist(), "keep_w": kw.round(3).tolist(),
        "alive": [bin(a) for a in al], "theta0": th[0].tolist() if len(th) else None, "lw": lw.round(1).tolist(),
        "est": e.round(2).tolist(), "truth": truth[k].round(2).tolist(),
        "trk_mean": [[float((x[j]*w[j]).sum()/w[j].sum()), float((y[j]*w[j]).sum()/w[j].sum())] for j in range(Tk)],
        "ess": pu.ess[:r.n_pairs].cpu().numpy().round(1).tolist(), "flags": pu.flags[:r.n_pairs].cpu().numpy().tolist()}))
