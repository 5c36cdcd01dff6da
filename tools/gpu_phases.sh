#!/bin/bash
# GPU parity tests, then the per-phase auction timeline (MUX_VERBOSE=1) with
# and without keeping the eps-CS assignment across phases.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for kc in 1 0; do
for sz in 4000 10000; do
  MUX_KEEP_CS=$kc MUX_VERBOSE=1 timeout 300 python bench.py --n $sz --m $sz --steps 2 --warmup 1 --no-cpu --no-e2e --no-mlp > gpurun_out/phases_kc${kc}_$sz.log 2>&1
done
done
