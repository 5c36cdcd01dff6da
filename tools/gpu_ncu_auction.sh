# ncu source-level profile of the auction kernel on a 2048 x 2048 round
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
CMD="python bench.py --n 2048 --m 2048 --steps 1 --warmup 1 --no-cpu --no-e2e"
$CMD > gpurun_out/plain_2k.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:auction_kernel -s 1 -c 1 -o gpurun_out/auction_2k $CMD > gpurun_out/ncu_2k.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_2k.log
echo finished
