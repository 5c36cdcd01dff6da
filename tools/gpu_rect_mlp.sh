cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
MUX_VERBOSE=1 timeout 900 python bench.py --n 10000 --m 40000 --steps 1 --warmup 0 --no-cpu --no-e2e --no-mlp > gpurun_out/rect_10k_40k.log 2>&1
echo "rect exit $?" >> gpurun_out/rect_10k_40k.log
python tools/mlp_only.py 2048 2048 > gpurun_out/mlp_plain.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mlp_pairs -s 1 -c 1 -o gpurun_out/mlp_v3_2k python tools/mlp_only.py 2048 2048 > gpurun_out/ncu_mlp.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_mlp.log
echo finished
