timeout 600 python -m pytest tests/test_gpu_pairs.py -q -x 2>&1 | tail -2
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-convoy 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); u=d['glmb_update']; print(' cfg3 update', round(u['ms'],3), u['stages_ms'])"
timeout 900 ncu --set full --clock-control none -k regex:'resample|reweight_cluster|assoc_sample' -c 3 -o gpurun_out/upd_full -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-convoy > /dev/null 2>&1
python profiles/ncu_summary.py gpurun_out/upd_full.ncu-rep > gpurun_out/upd_full_summary.txt 2>&1
