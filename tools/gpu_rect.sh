cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
MUX_VERBOSE=1 timeout 300 python bench.py --n 10000 --m 10000 --steps 1 --warmup 0 --no-cpu --no-e2e --no-mlp > gpurun_out/prof_10000.log 2>&1
MUX_VERBOSE=1 timeout 300 python bench.py --n 4000 --m 12000 --steps 1 --warmup 0 --no-cpu --no-e2e --no-mlp > gpurun_out/rect_4k_12k.log 2>&1
MUX_VERBOSE=1 timeout 300 python bench.py --n 12000 --m 4000 --steps 1 --warmup 0 --no-cpu --no-e2e --no-mlp > gpurun_out/rect_12k_4k.log 2>&1
MUX_VERBOSE=1 timeout 900 python bench.py --n 10000 --m 40000 --steps 1 --warmup 0 --no-cpu --no-e2e --no-mlp > gpurun_out/rect_10k_40k.log 2>&1
echo finished
