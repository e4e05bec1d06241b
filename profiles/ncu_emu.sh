set -u
mkdir -p gpurun_out
python -c "import sys; sys.path.insert(0,'.'); from paper_2512_06230_b200 import build; build.build()"
for E in -12 -6 0; do
  GLMB_COMPAT_K=2 GLMB_COMPAT_EMU=$E timeout 600 ncu --set full --clock-control none -k regex:compat -c 1 -o gpurun_out/emu${E} -f \
     python profiles/compat_sweep.py --child 3 2 > gpurun_out/emu${E}.log 2>&1
  python profiles/ncu_summary.py gpurun_out/emu${E}.ncu-rep > gpurun_out/emu${E}_summary.txt 2>&1
done
echo done
