#!/bin/bash
# full GPU suite (incl. the exchange-variant test), then an opt-in probe of concurrent long-path clusters with the push exchange
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_d.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_d.log
L=gpurun_out/conc_d.log; : > $L
MUX_SSP_CONC=4 N=2000 R=20 timeout 240 python tools/ssp_stress.py >> $L 2>&1; echo "conc stress exit $?" >> $L
for v in "MUX_SSP_CONC=4" "MUX_SSP_CONC=1"; do
  r=$(env $v timeout 240 python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e --no-mlp 2>gpurun_out/conc_d.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solver']; print(round(d['value'],2), [round(x,1) for x in d['ms_per_step_all']], 'dense', round(s['ms_dense'],1), s['dense_steps'], 'us/pop', round(1e3*s['ms_dense']/max(1,s['dense_steps']),3), 'tot', s['total_q'])")
  echo "$v: $r (exit $?)" >> $L
done
echo finished
