"""Per-seed convoy results for one cell (diagnostics): cardinality error, tracking error, and
the steps where the MAP cardinality departs from the truth."""
import json
import sys

import numpy as np

sys.path.insert(0, '.')
from paper_2512_06230_b200 import _lib
from paper_2512_06230_b200.build import build

build()
_lib.glmb_init(0)
from paper_2512_06230_b200.scenes import ConvoyConfig
from paper_2512_06230_b200.tracker import convoy_metrics, run_convoy

N = int(sys.argv[1]) if len(sys.argv) > 1 else 20
H = int(sys.argv[2]) if len(sys.argv) > 2 else 100
seeds = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else list(range(10))
extra = dict(a.split("=") for a in sys.argv[4].split(";")) if len(sys.argv) > 4 and sys.argv[4] else {}
def _conv(v):
    if "," in v:
        return tuple(float(x) for x in v.split(","))
    return float(v) if "." in v or "e" in v else int(v)


extra = {k: _conv(v) for k, v in extra.items()}
for seed in seeds:
    cfg = ConvoyConfig(N=N, H_max=H, seed=seed, **extra)
    recs, ests, truth = run_convoy(cfg, K_cap=4096)
    c, d = convoy_metrics(ests, truth)
    card = np.array([len(e) for e in ests]) - np.array([len(t) for t in truth])
    bad = np.nonzero(card)[0]
    print(json.dumps({"seed": seed, **extra, "card_err": round(c, 4), "track_err_m": round(d, 4),
                      "n_bad_steps": int(len(bad)), "first_bad": int(bad[0]) if len(bad) else None,
                      "card_diff_hist": {str(v): int((card == v).sum()) for v in np.unique(card)}}), flush=True)
