# quick GPU iteration: parity tests + bench at 1k / 4k / 10k (timers on)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for sz in 1000 4000; do
  MUX_VERBOSE=1 timeout 600 python bench.py --n $sz --m $sz --steps 2 --warmup 1 --no-cpu --no-e2e --no-mlp > gpurun_out/bench_$sz.log 2>&1
done
MUX_VERBOSE=1 timeout 600 python bench.py --n 10000 --m 10000 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_10000.log 2>&1
echo finished
