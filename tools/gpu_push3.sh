#!/bin/bash
# 512 vs 256-thread long-path CTAs: stress, A/B bench, GPU suite, then ncu of the default
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; L=gpurun_out/push3.log; : > $L
(timeout 300 python tools/ssp_stress.py; MUX_SSP_CT=256 R=20 timeout 300 python tools/ssp_stress.py) >> $L 2>&1
echo "stress exit $?" >> $L
for v in "MUX_SSP_CT=512" "MUX_SSP_CT=256" "MUX_SSP_CT=512" "MUX_SSP_CT=256"; do
  r=$(env $v timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e --no-mlp 2>gpurun_out/push3.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solver']; print(round(d['value'],2), [round(x,1) for x in d['ms_per_step_all']], 'dense', round(s['ms_dense'],1), s['dense_steps'], 'us/pop', round(1e3*s['ms_dense']/max(1,s['dense_steps']),3), 'par', round(s['ms_parallel'],2), 'tot', s['total_q'])")
  echo "$v: $r" >> $L
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_push3.log 2>&1
echo "pytest exit $?" >> $L
bash tools/gpu_ncu_push.sh
echo finished
