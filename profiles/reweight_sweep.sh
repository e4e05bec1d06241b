# cfg3 reweight / reweight_pairs standalone times and HBM fractions for GLMB_REWEIGHT_FLAT settings
# (default = e-cache; 1 = flat recompute, 2 = flat fp64 l-cache, 0 = cluster kernel)
for v in "$@"; do
  if [ "$v" = "def" ]; then unset GLMB_REWEIGHT_FLAT; else export GLMB_REWEIGHT_FLAT=$v; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-convoy --no-graphs --no-skip-probe 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('flat', '$v', 'reweight', round(d['stages_ms']['reweight'],4), 'frac', round(d['hbm_kernels']['reweight']['frac'],3), 'reweight_pairs', round(d['glmb_update']['stages_ms']['reweight_pairs'],4), round(d['glmb_update']['hbm_kernels']['reweight_pairs']['frac'],3), 'step', round(d['ms_per_step'],4))"
done
unset GLMB_REWEIGHT_FLAT
