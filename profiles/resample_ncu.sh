# ncu --set full of the cfg3 resample kernel (glmb_update in the bench), with source
timeout 900 ncu --set full --clock-control none --import-source on -k regex:resample -c 1 -o gpurun_out/res_full -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-convoy --no-graphs > gpurun_out/res_ncu.log 2>&1
echo "ncu exit $?"
python profiles/ncu_summary.py gpurun_out/res_full.ncu-rep > gpurun_out/res_full_summary.txt 2>&1
