#!/usr/bin/env bash
# The GPU-box recipe behind profiles/: parity tests, the bench line, the ncu launch list
# and one `ncu --set full` capture per hot kernel.  Run from the repo root under gpurun:
#   gpurun --timeout 1800 -- 'bash profiles/capture.sh r01'
# Outputs land in gpurun_out/ (scratch); the summaries worth keeping are copied to profiles/.
set -u
TAG=${1:-rXX}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $OUT/${TAG}_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/${TAG}_pytest_gpu.log 2>&1
echo "pytest_gpu exit $?"
tail -3 $OUT/${TAG}_pytest_gpu.log
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench exit $?"
cat $OUT/${TAG}_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
    > $OUT/${TAG}_ncu_list.log 2>&1
echo "ncu list exit $?"
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'compat|reweight|predict|birth' -c 8 -o $OUT/${TAG}_full -f \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/${TAG}_ncu_full.log 2>&1
echo "ncu full exit $?"
python profiles/ncu_summary.py $OUT/${TAG}_full.ncu-rep > $OUT/${TAG}_ncu_full_summary.txt 2>&1
echo done
