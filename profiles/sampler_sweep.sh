# cfg3 GLMB update: the update and assoc_sample times from the bench (repeat count as the argument)
for r in $(seq 1 ${1:-1}); do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-convoy --no-graphs --no-skip-probe 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); u=d['glmb_update']; print('update', round(u['ms'],4), 'one_call', round(u['one_call_ms'],4), 'assoc_sample', round(u['stages_ms']['assoc_sample'],4))"
done
