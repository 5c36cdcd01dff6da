#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/cl_sweep.log
(timeout 300 python tools/ssp_stress.py; N=3000 R=20 timeout 300 python tools/ssp_stress.py) >> gpurun_out/cl_sweep.log 2>&1
for cl in 8 4 16; do
  r=$(MUX_SSP_CL=$cl timeout 300 python bench.py --steps 6 --warmup 2 --no-cpu --no-e2e --no-mlp 2>gpurun_out/cl_$cl.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solver']; print(round(d['value'],2), [round(x,1) for x in d['ms_per_step_all']], 'dense', round(s['ms_dense'],1), s['dense_steps'], 'us/pop', round(1e3*s['ms_dense']/max(1,s['dense_steps']),3))")
  echo "cluster $cl: $r" >> gpurun_out/cl_sweep.log
done
echo finished
