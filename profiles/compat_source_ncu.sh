# source-level ncu of one cfg3 compat launch (round-2 starting point): per-line instructions and stall samples
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'compat_kernel' -s 3 -c 1 -o gpurun_out/compat_src -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-update --no-convoy --no-graphs --no-skip-probe > gpurun_out/compat_src.log 2>&1
echo "ncu exit $?"
