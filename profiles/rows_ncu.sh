timeout 900 ncu --set full --clock-control none --import-source on -k regex:'rows_fill|rows_count' -s 200 -c 2 -o gpurun_out/rows_full -f python profiles/convoy_run.py 120 > gpurun_out/rows_ncu.log 2>&1
echo "ncu exit $?"
python profiles/ncu_summary.py gpurun_out/rows_full.ncu-rep > gpurun_out/rows_full_summary.txt 2>&1
