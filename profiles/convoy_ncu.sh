# ncu --set full of the convoy's sampler / pairs / prune kernels at a late step (N=20, H_max=100)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'assoc_sample|prune|invert|number|row_count|first' -s 600 -c 6 -o gpurun_out/conv_full -f python profiles/convoy_profile.py 120 > gpurun_out/conv_ncu.log 2>&1
echo "ncu exit $?"
python profiles/ncu_summary.py gpurun_out/conv_full.ncu-rep > gpurun_out/conv_full_summary.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/conv_launches.csv python profiles/convoy_profile.py 120 > /dev/null 2>&1
python profiles/launch_summary.py gpurun_out/conv_launches.csv > gpurun_out/conv_launch_summary.txt 2>&1
echo done
