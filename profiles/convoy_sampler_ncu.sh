# ncu --set full of the convoy's two-stage sampler (N = 20, H_max = 100, count prior) at a late update
cat > gpurun_out/convoy_run.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch
from paper_2512_06230_b200 import _lib as L
from paper_2512_06230_b200.scenes import ConvoyConfig
from paper_2512_06230_b200.tracker import run_convoy
torch.cuda.set_device(0); L.glmb_init(0)
recs, _, _ = run_convoy(ConvoyConfig(N=20, H_max=100, K=90), K_cap=4096, with_estimates=False)
print("T_k", recs[-1].T_k, "M", recs[-1].M, "parents", recs[-1].n_parents, "pairs", recs[-1].n_pairs)
PY
python gpurun_out/convoy_run.py
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'assoc_sample' -s 85 -c 1 -o gpurun_out/csamp_full -f python gpurun_out/convoy_run.py > /dev/null 2>&1
python profiles/ncu_summary.py gpurun_out/csamp_full.ncu-rep > gpurun_out/csamp_full_summary.txt 2>&1
python profiles/cuda_line_hotspots.py gpurun_out/csamp_full.ncu-rep 40 > gpurun_out/csamp_lines.txt 2>&1
echo done
