#!/usr/bin/env bash
# The GPU-box recipe behind profiles/: parity tests, the bench line, the ncu launch list
# and `ncu --set full` captures of the step kernels and of the GLMB-update kernels, with
# per-line hot spots of the dominant ones.  Run from the repo root under gpurun:
#   gpurun --timeout 3000 -- 'bash profiles/capture.sh r02a'
# Outputs land in gpurun_out/ (scratch); the summaries worth keeping are copied to profiles/.
set -u
TAG=${1:-rXX}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $OUT/${TAG}_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest_gpu exit $?"
tail -3 $OUT/${TAG}_pytest_gpu.log
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench exit $?"
timeout 900 python bench.py --impl reference > $OUT/${TAG}_bench_ref.json 2> $OUT/${TAG}_bench_ref.err
echo "bench reference exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
    --no-convoy --no-graphs --no-skip-probe --no-b2b > $OUT/${TAG}_ncu_list.log 2>&1
echo "ncu list exit $?"
python profiles/launch_summary.py $OUT/${TAG}_launches.csv > $OUT/${TAG}_launch_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'compat_kernel|reweight_ecache|predict|birth' -s 8 -c 4 -o $OUT/${TAG}_full -f \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-convoy --no-graphs --no-skip-probe --no-b2b \
    --no-update > $OUT/${TAG}_ncu_full.log 2>&1
echo "ncu full exit $?"
python profiles/ncu_summary.py $OUT/${TAG}_full.ncu-rep > $OUT/${TAG}_ncu_full_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'assoc_sample|resample_kernel|prune_kernel|invert_kernel|dedup_kernel|rows_fill|death_prob' \
    -s 14 -c 7 -o $OUT/${TAG}_upd -f \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-convoy --no-graphs --no-skip-probe --no-b2b \
    > $OUT/${TAG}_ncu_upd.log 2>&1
echo "ncu update exit $?"
# reweight_pairs (the e-cache kernel in pair mode): the first launch after the step's 9 theta-mode ones
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'reweight_ecache' -s 10 -c 1 \
    -o $OUT/${TAG}_rwp -f python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-convoy \
    --no-graphs --no-skip-probe > $OUT/${TAG}_ncu_rwp.log 2>&1
echo "ncu reweight_pairs exit $?"
python profiles/ncu_summary.py $OUT/${TAG}_upd.ncu-rep $OUT/${TAG}_rwp.ncu-rep > $OUT/${TAG}_ncu_update_summary.txt 2>&1
for k in full upd; do
  python profiles/cuda_line_hotspots.py $OUT/${TAG}_${k}.ncu-rep 25 > $OUT/${TAG}_${k}_lines.txt 2>&1
done
echo done
