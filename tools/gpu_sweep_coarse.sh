#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/sweep_coarse.log
for cp in 0 2000 800 300 100; do
  r=$(MUX_SSP_COARSE_POPS=$cp timeout 300 python bench.py --steps 4 --warmup 2 --no-cpu --no-e2e --no-mlp 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solver']; print(round(d['value'],2), [round(x,1) for x in d['ms_per_step_all']], 'dense', round(s['ms_dense'],1), s['dense_steps'], 'par', round(s['ms_parallel'],1), s['dense_searches'], 'match', round(s['ms_match'],1))")
  echo "coarse_pops $cp: $r" >> gpurun_out/sweep_coarse.log
done
MUX_SSP_COARSE_POPS=300 MUX_VERBOSE=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-mlp > /dev/null 2> gpurun_out/verbose_coarse.err
echo finished
