# A/B of compat's unit order (tile-major vs track-major) at cfg3: time and DRAM traffic
for O in 0 1; do
  GLMB_COMPAT_ORDER=$O python profiles/compat_sweep.py --reps 20 2,-10 2>&1 | tail -1
  GLMB_COMPAT_ORDER=$O timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:compat -c 1 python profiles/compat_sweep.py --child 3 1 2>&1 | grep -E "dram__bytes_read|gpu__time" 
done
