# ncu --set full of the cfg3 two-stage sampler (glmb_update in the bench) on the bench's timed C_k
# (after the warm-up steps' predicts), with source; then the per-line hot spots
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-convoy --no-graphs --no-skip-probe 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); u=d['glmb_update']; print(' cfg3 update', round(u['ms'],3), u['stages_ms'], u['n_kept'], u['n_unique'], u['gated_entries'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'assoc_sample' -s 4 -c 1 -o gpurun_out/samp_full -f python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-convoy --no-graphs --no-skip-probe > /dev/null 2>&1
python profiles/ncu_summary.py gpurun_out/samp_full.ncu-rep > gpurun_out/samp_full_summary.txt 2>&1
python profiles/cuda_line_hotspots.py gpurun_out/samp_full.ncu-rep 40 > gpurun_out/samp_lines.txt 2>&1
echo done
