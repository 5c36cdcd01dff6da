# tests + MLP/auction bench at 10k, then the 2-GPU checks (run with gpurun --gpus 2)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
MUX_VERBOSE=1 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_10000.log 2>&1
bash tools/gpu_multi.sh
echo finished
