# ncu: MLP kernel (full set), auction kernel at 4k (full set), launch list of one bench step
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python tools/mlp_only.py 2048 2048 > gpurun_out/mlp_plain.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mlp_pairs -s 1 -c 1 -o gpurun_out/mlp_2k python tools/mlp_only.py 2048 2048 > gpurun_out/ncu_mlp.log 2>&1
echo "ncu mlp exit $?" >> gpurun_out/ncu_mlp.log
CMD="python bench.py --n 4000 --m 4000 --steps 1 --warmup 1 --no-cpu --no-e2e --no-mlp"
$CMD > gpurun_out/plain_4k.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:auction_kernel -s 1 -c 1 -o gpurun_out/auction_4k $CMD > gpurun_out/ncu_auction.log 2>&1
echo "ncu auction exit $?" >> gpurun_out/ncu_auction.log
CMD2="python bench.py --n 10000 --m 10000 --steps 1 --warmup 1 --no-cpu --no-e2e"
$CMD2 > gpurun_out/plain_10k.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_10k.csv $CMD2 > gpurun_out/ncu_launches.log 2>&1
echo "ncu launches exit $?" >> gpurun_out/ncu_launches.log
echo finished
