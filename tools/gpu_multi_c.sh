#!/bin/bash
# 2-GPU box: N=1 and N=2 (replicas, torchrun) bench lines with the current long-path kernel, sharded scoring check
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu > gpurun_out/bench_1gpu_c.json 2> gpurun_out/bench_1gpu_c.err
timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_2gpu_c.json 2> gpurun_out/bench_2gpu_c.err
echo "bench2 exit $?" >> gpurun_out/bench_2gpu_c.err
timeout 600 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/sharded_check.py 2000 > gpurun_out/sharded_check_c.log 2>&1
echo "sharded exit $?" >> gpurun_out/sharded_check_c.log
echo finished
