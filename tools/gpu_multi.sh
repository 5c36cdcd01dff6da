# 2-GPU checks: row-sharded round vs single GPU, and the bench under torchrun
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 600 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/sharded_check.py 2000 > gpurun_out/sharded_check.log 2>&1
echo "sharded exit $?" >> gpurun_out/sharded_check.log
timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_2gpu.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_2gpu.log
echo finished
