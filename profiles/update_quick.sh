# cfg3 GLMB update stage times (bench) and the convoy (3 seeds) per-update time and stages
bash profiles/sampler_sweep.sh 2
python -c "
import sys; sys.path.insert(0,'.')
import bench, torch
dev=torch.device('cuda',0); torch.cuda.set_device(0)
from paper_2512_06230_b200 import _lib as L; L.glmb_init(0)
c=bench.bench_convoy(dev, seeds=range(3)); print('convoy', round(c['update_ms_mean'],3), round(c['device_ms_mean'],3), {k: round(v,4) for k,v in c['stages_ms'].items()})
"
