cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --n 1000 --m 1000 --steps 3 --warmup 1 --no-cpu > gpurun_out/bench1k.log 2>&1
timeout 400 python bench.py --n 4000 --m 4000 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench4k.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/bench10k.log 2>&1
echo finished
