#!/bin/bash
# GPU parity tests + default bench + a verbose 10k breakdown
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
MUX_VERBOSE=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-mlp > gpurun_out/bench_verbose.json 2> gpurun_out/bench_verbose.err
echo finished
