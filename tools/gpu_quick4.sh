#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
MUX_VERBOSE=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-mlp > gpurun_out/bench_verbose.json 2> gpurun_out/bench_verbose.err
echo finished
