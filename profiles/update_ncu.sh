# ncu --set full of the GLMB-update kernels at cfg3 (one launch each) -> a summary for profiles/
timeout 1200 ncu --set full --clock-control none -k regex:'assoc_sample|resample_kernel|reweight_flat|prune_kernel|invert_kernel|dedup_kernel|rows_fill|death_prob' -c 12 -o gpurun_out/upd_full -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-convoy --no-graphs --no-skip-probe > gpurun_out/upd_ncu.log 2>&1
echo "ncu exit $?"
python profiles/ncu_summary.py gpurun_out/upd_full.ncu-rep > gpurun_out/upd_full_summary.txt 2>&1
