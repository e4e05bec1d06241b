# A/B of the sampler's samples-per-CTA on the cfg3 GLMB update and the convoy (diagnostics)
for S in 0 1 2 4 8 16; do
  echo "spc=$S"
  GLMB_SAMPLES_PER_CTA=$S timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-convoy 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); u=d['glmb_update']; print(' cfg3 update', round(u['ms'],3), 'sample', round(u['stages_ms']['assoc_sample'],3))"
  GLMB_SAMPLES_PER_CTA=$S timeout 300 python profiles/convoy_grid.py 20 100 2>/dev/null | tail -1
done
