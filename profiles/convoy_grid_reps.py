"""The paper's convoy protocol: grid N x H_max, R repetitions per
cell (seeds 0..R-1: new detections and filter draws each run), 548 steps per run.
One JSON line per cell: mean +- SEM over the runs of the MAP cardinality error, the
Hungarian tracking error and the per-update wall / device time (methodology M3)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, '.')
from paper_2512_06230_b200 import _lib
from paper_2512_06230_b200.build import build

build()
_lib.glmb_init(0)
from paper_2512_06230_b200.scenes import ConvoyConfig
from paper_2512_06230_b200.tracker import convoy_metrics, run_convoy

Ns = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 2, 5, 10, 20]
Hs = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [5, 10, 25, 50, 100]
R = int(sys.argv[3]) if len(sys.argv) > 3 else 10


def ms(a):
    a = np.asarray(a, np.float64)
    return [round(float(a.mean()), 5), round(float(a.std(ddof=1) / np.sqrt(len(a))) if len(a) > 1 else 0.0, 5)]


run_convoy(ConvoyConfig(N=2, H_max=10, K=20), K_cap=256)   # warm-up (module load, allocator)
for N in Ns:
    for H in Hs:
        card, dist, upd, dev = [], [], [], []
        t0 = time.time()
        for seed in range(R):
            cfg = ConvoyConfig(N=N, H_max=H, seed=seed)
            recs, ests, truth = run_convoy(cfg, K_cap=4096)
            c, d = convoy_metrics(ests, truth)
            card.append(c)
            dist.append(d)
            upd.append(np.mean([r.wall_ms for r in recs]))
            dev.append(np.mean([r.device_ms for r in recs]))
        print(json.dumps({"N": N, "H_max": H, "runs": R, "card_err": ms(card), "track_err_m": ms(dist),
                          "update_ms": ms(upd), "device_ms": ms(dev), "cell_s": round(time.time() - t0, 1)}),
              flush=True)
