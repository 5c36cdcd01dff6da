#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/conc2.log
MUX_SSP_CONC=1 R=10 timeout 120 python tools/ssp_stress.py >> gpurun_out/conc2.log 2>&1; echo "conc1 rc $?" >> gpurun_out/conc2.log
MUX_SSP_CONC=4 R=10 timeout 120 python -X faulthandler tools/ssp_stress.py >> gpurun_out/conc2.log 2>&1; echo "conc4 rc $?" >> gpurun_out/conc2.log
for seed in 0 1 2; do
  MUX_SSP_CONC=4 MUX_VERBOSE=1 timeout 60 python -c "
import os,sys; sys.path.insert(0,'.')
from paper_2303_13803_b200 import default_table
from paper_2303_13803_b200.scheduler import round_arrays
from paper_2303_13803_b200.synth import make_cluster
cl=make_cluster(2000,2000,seed=$seed); print(round_arrays(default_table(), cl.x, cl.share, cl.y, qbits=30)[1])
" > gpurun_out/conc2_seed$seed.log 2>&1; echo "seed $seed rc $?" >> gpurun_out/conc2.log
done
echo finished
