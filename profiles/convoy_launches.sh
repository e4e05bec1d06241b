# per-kernel device time of 120 convoy updates (ncu launch list, serialised) + the un-profiled device time
timeout 600 python -c "
import sys, statistics; sys.path.insert(0, '.')
from paper_2512_06230_b200 import _lib
from paper_2512_06230_b200.build import build
build(); _lib.glmb_init(0)
from paper_2512_06230_b200.scenes import ConvoyConfig
from paper_2512_06230_b200.tracker import run_convoy
run_convoy(ConvoyConfig(N=20, H_max=100, K=40), K_cap=4096, with_estimates=False)
recs, _, _ = run_convoy(ConvoyConfig(N=20, H_max=100, K=120), K_cap=4096, with_estimates=False)
print('device ms/update (updates 1..120):', statistics.mean(r.device_ms for r in recs[1:]), 'wall', statistics.mean(r.wall_ms for r in recs[1:]))
"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/conv_launches.csv python profiles/convoy_run.py 120 > /dev/null 2>&1
python profiles/launch_summary.py gpurun_out/conv_launches.csv > gpurun_out/conv_launch_summary.txt 2>&1
