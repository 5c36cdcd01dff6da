#!/bin/bash
mkdir -p gpurun_out
for q in 30 24 16; do
MUX_VERBOSE=1 timeout 300 python bench.py --n 10000 --m 10000 --qbits $q --steps 4 --warmup 1 --no-cpu --no-e2e --no-mlp > gpurun_out/q_$q.log 2>&1
done
