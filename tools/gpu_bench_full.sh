# the driver's round-end commands: default bench (N=1) and the reference arm
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_default.log
timeout 1200 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1
echo "ref exit $?" >> gpurun_out/bench_reference.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
echo finished
