#!/bin/bash
# round-1 (third session) evidence: default bench (with CPU baseline + e2e), reference arm, ncu full set of
# every long-path cluster launch of one 10k solve (traffic), launch list of one bench step, smoke
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_c.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_c.log
timeout 600 python bench.py > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; echo "bench exit $?" >> gpurun_out/bench_c.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_c.json 2> gpurun_out/bench_ref_c.err
timeout 300 python tools/ssp_one.py 10000 > gpurun_out/one_10k_c.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:ssp_cluster_kernel -o gpurun_out/ssp_cluster_all_c python tools/ssp_one.py 10000 > gpurun_out/ncu_cluster_all_c.log 2>&1
echo "ncu cluster exit $?" >> gpurun_out/ncu_cluster_all_c.log
CMD2="python bench.py --n 10000 --m 10000 --steps 1 --warmup 1 --no-cpu --no-e2e --no-mlp"
$CMD2 > gpurun_out/plain_10k_c.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_10k_c.csv $CMD2 > gpurun_out/ncu_launches_c.log 2>&1
echo "ncu launches exit $?" >> gpurun_out/ncu_launches_c.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-mlp > gpurun_out/bench_c2.json 2>> gpurun_out/bench_c.err
echo finished
