# cfg3 reweight (theta mode): standalone times of the flat kernel variants (GLMB_REWEIGHT_FLAT = 1 recompute,
# 2 l-cache) from the bench's serialised stage pass, then ncu --set full of the default with per-line hot spots
for v in; do
  GLMB_REWEIGHT_FLAT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-convoy --no-graphs --no-skip-probe 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('flat', '$v', 'reweight', round(d['stages_ms']['reweight'],4), 'frac', round(d['hbm_kernels']['reweight']['frac'],3), 'reweight_pairs', round(d['glmb_update']['stages_ms']['reweight_pairs'],4), round(d['glmb_update']['hbm_kernels']['reweight_pairs']['frac'],3))"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'reweight_tma|reweight_ecache|reweight_flat' -s 3 -c 1 -o gpurun_out/rw_full -f python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-convoy --no-graphs --no-skip-probe --no-update > /dev/null 2>&1
python profiles/ncu_summary.py gpurun_out/rw_full.ncu-rep > gpurun_out/rw_full_summary.txt 2>&1
python profiles/cuda_line_hotspots.py gpurun_out/rw_full.ncu-rep 40 > gpurun_out/rw_lines.txt 2>&1
echo done
