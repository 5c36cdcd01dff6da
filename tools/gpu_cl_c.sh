#!/bin/bash
# cluster size with the push exchange: 8 (512 threads, default) vs 16 / 4 (1024 threads)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; L=gpurun_out/cl_c.log; : > $L
(MUX_SSP_CL=16 N=2000 R=20 timeout 300 python tools/ssp_stress.py; MUX_SSP_CL=4 N=2000 R=20 timeout 300 python tools/ssp_stress.py) >> $L 2>&1
echo "stress exit $?" >> $L
for rep in 1 2; do
for v in "MUX_SSP_CL=8" "MUX_SSP_CL=16" "MUX_SSP_CL=4"; do
  r=$(env $v timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e --no-mlp 2>gpurun_out/cl_c.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solver']; print(round(d['value'],2), [round(x,1) for x in d['ms_per_step_all']], 'dense', round(s['ms_dense'],1), s['dense_steps'], 'us/pop', round(1e3*s['ms_dense']/max(1,s['dense_steps']),3), 'par', round(s['ms_parallel'],2), 'tot', s['total_q'])")
  echo "$v: $r" >> $L
done
done
echo finished
