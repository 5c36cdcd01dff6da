cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
: > gpurun_out/sweep2.txt
for sz in 4000 10000; do for T in 16 32 64 128 256; do
  MUX_TAIL=$T MUX_VERBOSE=1 timeout 300 python bench.py --n $sz --m $sz --steps 1 --warmup 0 --no-cpu --no-e2e --no-mlp > gpurun_out/sw.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]);s=d['solver'];print('n=$sz T=$T', round(d['value'],1), s['rounds'], s['tail_bids'], round(s['ms_tail'],1))" >> gpurun_out/sweep2.txt 2>&1
  grep "rejected" gpurun_out/sw.log | tail -1 >> gpurun_out/sweep2.txt
done; done
echo finished
