#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
(timeout 300 python tools/ssp_stress.py; N=3000 R=20 timeout 300 python tools/ssp_stress.py; N=1000 Q=20 R=30 timeout 300 python tools/ssp_stress.py) > gpurun_out/stress.log 2>&1
timeout 300 python bench.py --steps 6 --warmup 2 --no-cpu --no-e2e --no-mlp > gpurun_out/bench_sq.json 2>/dev/null
timeout 600 python -m pytest tests/test_gpu_ssp.py -q -x > gpurun_out/pytest_ssp.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_ssp.log
echo finished
