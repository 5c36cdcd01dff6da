#!/bin/bash
# GPU parity tests (incl. tie canonicalisation), then round timings with the
# canonicalisation statistics.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for sz in 4000 10000; do
  MUX_VERBOSE=1 timeout 300 python bench.py --n $sz --m $sz --steps 2 --warmup 1 --no-cpu --no-e2e --no-mlp > gpurun_out/canon_$sz.log 2>&1
done
MUX_VERBOSE=1 timeout 300 python bench.py --n 5000 --m 20000 --steps 1 --warmup 1 --no-cpu --no-e2e --no-mlp > gpurun_out/canon_5k20k.log 2>&1
