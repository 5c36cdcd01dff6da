# (K, theta) sweep at 10k over two seeds: auction kernel time only
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/sweep.txt
for seed in 0 1; do for k in 8 15; do for th in 4 6; do
  MUX_K=$k MUX_THETA=$th timeout 300 python bench.py --n 10000 --m 10000 --steps 1 --warmup 0 --seed $seed --no-cpu --no-e2e --no-mlp > gpurun_out/sw.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]);s=d['solver'];print('seed=$seed K=$k th=$th', round(d['value'],1), s['rounds'], s['tail_bids'], s['row_scans'])" >> gpurun_out/sweep.txt 2>&1
done; done; done
echo finished
