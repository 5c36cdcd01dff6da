#!/bin/bash
# ncu of the push-exchange long-path kernel (full set + source) and the launch list of one bench step
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/ssp_one.py 10000 > gpurun_out/one_10k.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ssp_cluster_kernel -c 2 -o gpurun_out/ssp_cluster_push python tools/ssp_one.py 10000 > gpurun_out/ncu_cluster_push.log 2>&1
echo "ncu cluster exit $?" >> gpurun_out/ncu_cluster_push.log
CMD2="python bench.py --n 10000 --m 10000 --steps 1 --warmup 1 --no-cpu --no-e2e"
$CMD2 > gpurun_out/plain_10k.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_10k.csv $CMD2 > gpurun_out/ncu_launches.log 2>&1
echo "ncu launches exit $?" >> gpurun_out/ncu_launches.log
echo finished
