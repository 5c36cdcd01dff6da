# auction timing breakdown (MUX_VERBOSE prints tail / round / scan-stage timers)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
MUX_VERBOSE=1 timeout 600 python bench.py --n 2048 --m 2048 --steps 1 --warmup 1 --no-cpu --no-e2e --no-mlp > gpurun_out/prof_2048.log 2>&1
MUX_VERBOSE=1 timeout 600 python bench.py --n 10000 --m 10000 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/prof_10000.log 2>&1
MUX_CG_SYNC=1 MUX_VERBOSE=1 timeout 600 python bench.py --n 10000 --m 10000 --steps 1 --warmup 1 --no-cpu --no-e2e --no-mlp > gpurun_out/prof_10000_cg.log 2>&1
echo finished
