"""Tracker-quality sweep on the paper-shaped convoy (diagnostics): one JSON line per setting."""
import sys, json, time
sys.path.insert(0, '.')
import numpy as np
from paper_2512_06230_b200 import _lib
from paper_2512_06230_b200.build import build
build(); _lib.glmb_init(0)
from paper_2512_06230_b200.scenes import ConvoyConfig
from paper_2512_06230_b200.tracker import run_convoy, convoy_metrics
base = dict(N=20, K=150)
settings = [dict(), dict(r_birth=0.5), dict(P=2048), dict(sigma_a=1.0, sigma_w=0.5), dict(sigma_a=4.0, sigma_w=2.0),
            dict(count_prior=False), dict(p_s=0.999), dict(birth_cov=(0.05, 0.05, 0.5, 0.05, 0.05)), dict(H_up=300)]
for st in settings:
    cfg = ConvoyConfig(**{**base, **st})
    t0 = time.time()
    recs, ests, truth = run_convoy(cfg, K_cap=2048)
    warm = cfg.N * cfg.delta + 10
    card, dist = convoy_metrics(ests[warm:], truth[warm:])
    dev = np.array([r.device_ms for r in recs])
    print(json.dumps({"setting": {k: v for k, v in st.items()}, "card_err": round(card, 4), "track_err_m": round(dist, 4),
                      "dev_ms": round(float(dev[5:].mean()), 3), "card_last": len(ests[-1])}), flush=True)
