"""The paper's convoy grid: N x H_max (+ the count-prior switch), full 548 steps.
One JSON line per cell: MAP cardinality error, Hungarian tracking error, per-update times."""
import sys, json, time
sys.path.insert(0, '.')
import numpy as np
from paper_2512_06230_b200 import _lib
from paper_2512_06230_b200.build import build
build(); _lib.glmb_init(0)
from paper_2512_06230_b200.scenes import ConvoyConfig
from paper_2512_06230_b200.tracker import run_convoy, convoy_metrics
Ns = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 2, 5, 10, 20]
Hs = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [100]
extra = [dict(a.split("=") for a in arg.split(";")) if arg else {} for arg in (sys.argv[3].split("|") if len(sys.argv) > 3 else [""])]
for ex in extra:
    def conv(v):
        if v in ("True", "False"):
            return v == "True"
        try:
            return float(v) if "." in v else int(v)
        except ValueError:
            return v
    ex = {k: conv(v) for k, v in ex.items()}
    for N in Ns:
        for H in Hs:
            cfg = ConvoyConfig(N=N, H_max=H, **ex)
            t0 = time.time()
            recs, ests, truth = run_convoy(cfg, K_cap=4096)
            wall = time.time() - t0
            card, dist = convoy_metrics(ests, truth)
            dev = np.array([r.device_ms for r in recs]); wl = np.array([r.wall_ms for r in recs])
            print(json.dumps({"N": N, "H_max": H, **ex, "card_err": round(card, 4), "track_err_m": round(dist, 4),
                              "update_ms_mean": round(float(wl.mean()), 3), "update_ms_p95": round(float(np.percentile(wl, 95)), 3),
                              "device_ms_mean": round(float(dev.mean()), 3), "pairs_max": max(r.n_pairs for r in recs),
                              "run_s": round(wall, 2)}), flush=True)
