#!/bin/bash
# Round-end evidence: GPU parity tests, smoke, default bench (+ reference arm),
# ncu launch list of one bench step, ncu --set full of the solver kernels.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-mlp"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_10k.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "ncu launches exit $?" >> gpurun_out/ncu_launches.log
python tools/ssp_one.py > gpurun_out/ssp_one.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ssp_cluster_kernel -c 12 -o gpurun_out/ssp_cluster_10k python tools/ssp_one.py > gpurun_out/ncu_cluster.log 2>&1
echo "ncu cluster exit $?" >> gpurun_out/ncu_cluster.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ssp_parallel_kernel -c 3 -o gpurun_out/ssp_parallel_10k python tools/ssp_one.py > gpurun_out/ncu_par.log 2>&1
echo "ncu parallel exit $?" >> gpurun_out/ncu_par.log
echo finished
