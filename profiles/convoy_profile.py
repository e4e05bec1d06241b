"""Per-kernel device time of the convoy update (N=20, H_max=100): a short run for ncu's launch list."""
import sys
sys.path.insert(0, '.')
from paper_2512_06230_b200 import _lib
from paper_2512_06230_b200.build import build
build(); _lib.glmb_init(0)
from paper_2512_06230_b200.scenes import ConvoyConfig
from paper_2512_06230_b200.tracker import run_convoy
run_convoy(ConvoyConfig(N=20, H_max=100, K=int(sys.argv[1]) if len(sys.argv) > 1 else 80), K_cap=4096, with_estimates=False)
