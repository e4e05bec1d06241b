import sys, time, json
sys.path.insert(0, '.')
import numpy as np
from paper_2512_06230_b200 import _lib
from paper_2512_06230_b200.build import build
build(); _lib.glmb_init(0)
from paper_2512_06230_b200.scenes import ConvoyConfig
from paper_2512_06230_b200.tracker import run_convoy, convoy_metrics
for N, H in [(3, 20), (5, 25), (20, 100)]:
    cfg = ConvoyConfig(N=N, H_max=H, K=548 if N == 20 else 150)
    t0 = time.time()
    recs, ests, truth = run_convoy(cfg, K_cap=2048)
    dt = time.time() - t0
    warm = N * cfg.delta + 10
    card, dist = convoy_metrics(ests[warm:], truth[warm:])
    dev = np.array([r.device_ms for r in recs]); wall = np.array([r.wall_ms for r in recs])
    print(json.dumps({"N": N, "H_max": H, "steps": len(recs), "total_s": dt, "card_err": card, "track_err_m": dist,
          "dev_ms_mean": dev[5:].mean(), "dev_ms_p95": float(np.percentile(dev[5:], 95)), "wall_ms_mean": wall[5:].mean(),
          "pairs_max": max(r.n_pairs for r in recs), "kept_mean": float(np.mean([r.n_kept for r in recs])),
          "card_last": [len(e) for e in ests[-5:]], "truth_last": len(truth[-1])}), flush=True)
