#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 1500 python tools/replay.py > gpurun_out/replay.json 2> gpurun_out/replay.err
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-mlp"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_10k.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo finished
