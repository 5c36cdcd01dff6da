# parity tests + 10k bench across epsilon-scaling factors
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for th in 4 6 8; do
  MUX_THETA=$th MUX_VERBOSE=1 timeout 600 python bench.py --n 10000 --m 10000 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/theta_$th.log 2>&1
done
MUX_THETA=4 MUX_VERBOSE=1 timeout 600 python bench.py --n 4000 --m 4000 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/theta4_4k.log 2>&1
MUX_THETA=4 MUX_VERBOSE=1 timeout 600 python bench.py --n 1000 --m 1000 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/theta4_1k.log 2>&1
echo finished
