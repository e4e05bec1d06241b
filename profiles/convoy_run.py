#!/usr/bin/env python
"""K convoy updates (N = 20, H_max = 100) through ConvoyTracker -- the process the convoy ncu
scripts profile.  usage: python profiles/convoy_run.py [K]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_06230_b200 import _lib  # noqa: E402
from paper_2512_06230_b200.build import build  # noqa: E402
from paper_2512_06230_b200.scenes import ConvoyConfig  # noqa: E402
from paper_2512_06230_b200.tracker import run_convoy  # noqa: E402

build()
_lib.glmb_init(0)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 120
run_convoy(ConvoyConfig(N=20, H_max=100, K=K), K_cap=4096, with_estimates=False)
