#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/sweep_budget.log
for sb in 192 96 48 24; do for db in 8 4 2; do
  r=$(MUX_SSP_STEPS=$sb MUX_SSP_DEEP=$db timeout 300 python bench.py --steps 4 --warmup 2 --no-cpu --no-e2e --no-mlp 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solver']; print(round(d['value'],2), [round(x,1) for x in d['ms_per_step_all']], 'dense', round(s['ms_dense'],1), s['dense_steps'], 'par', round(s['ms_parallel'],1), s['dense_searches'])")
  echo "steps $sb deep $db: $r" >> gpurun_out/sweep_budget.log
done; done
echo finished
