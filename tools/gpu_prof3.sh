cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for sz in 4000 10000; do
MUX_VERBOSE=1 timeout 600 python bench.py --n $sz --m $sz --steps 3 --warmup 1 --no-cpu --no-e2e --no-mlp > gpurun_out/prof_$sz.log 2>&1
done
echo finished
