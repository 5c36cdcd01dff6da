#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/conc_sweep.log
(timeout 300 python tools/ssp_stress.py; N=3000 R=20 timeout 300 python tools/ssp_stress.py; N=4000 R=6 timeout 300 python tools/ssp_stress.py) >> gpurun_out/conc_sweep.log 2>&1
for c in 1 2 4 8; do
  r=$(MUX_SSP_CONC=$c timeout 300 python bench.py --steps 6 --warmup 2 --no-cpu --no-e2e --no-mlp 2>gpurun_out/conc_$c.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solver']; print(round(d['value'],2), [round(x,1) for x in d['ms_per_step_all']], 'dense', round(s['ms_dense'],1), s['dense_steps'], s['dense_searches'])")
  echo "conc $c: $r" >> gpurun_out/conc_sweep.log
done
MUX_VERBOSE=1 MUX_SSP_CONC=4 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-mlp > /dev/null 2> gpurun_out/conc_verbose.err
echo finished
