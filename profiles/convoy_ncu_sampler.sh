timeout 900 ncu --set full --clock-control none --import-source on -k regex:'assoc_sample' -s 100 -c 1 -o gpurun_out/conv_samp -f python profiles/convoy_profile.py 120 > gpurun_out/conv_ncu.log 2>&1
echo "ncu exit $?"
python profiles/ncu_summary.py gpurun_out/conv_samp.ncu-rep > gpurun_out/conv_samp_summary.txt 2>&1
