# ncu --set full of the cfg3 two-stage sampler (glmb_update in the bench), with source
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-convoy 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); u=d['glmb_update']; print(' cfg3 update', round(u['ms'],3), u['stages_ms'], u['n_kept'], u['n_unique'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'assoc_sample' -c 2 -o gpurun_out/samp_full -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-convoy > /dev/null 2>&1
python profiles/ncu_summary.py gpurun_out/samp_full.ncu-rep > gpurun_out/samp_full_summary.txt 2>&1
ncu -i gpurun_out/samp_full.ncu-rep --page source --csv > gpurun_out/samp_source.csv 2>&1
echo done
