# auction timing breakdown at 4k and 10k (MUX_VERBOSE prints tail stats)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for sz in 4000 10000; do
  MUX_VERBOSE=1 timeout 600 python bench.py --n $sz --m $sz --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/prof_$sz.log 2>&1
done
echo finished
