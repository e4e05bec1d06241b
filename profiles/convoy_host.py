"""Host-side cost of the convoy update loop (cProfile over 200 updates, N=20, H_max=100)."""
import cProfile
import pstats
import sys
sys.path.insert(0, '.')
from paper_2512_06230_b200 import _lib
from paper_2512_06230_b200.build import build
build(); _lib.glmb_init(0)
from paper_2512_06230_b200.scenes import ConvoyConfig
from paper_2512_06230_b200.tracker import run_convoy
run_convoy(ConvoyConfig(N=20, H_max=100, K=40), K_cap=4096, with_estimates=False)
pr = cProfile.Profile()
pr.enable()
recs, _, _ = run_convoy(ConvoyConfig(N=20, H_max=100, K=200), K_cap=4096, with_estimates=False)
pr.disable()
import statistics
print("wall ms", statistics.mean(r.wall_ms for r in recs[50:]), "device ms", statistics.mean(r.device_ms for r in recs[50:]))
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
