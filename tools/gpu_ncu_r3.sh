mkdir -p gpurun_out/r3ncu3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3ncu3/build.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-mlp --no-schedule > gpurun_out/r3ncu3/bench.json 2> gpurun_out/r3ncu3/bench.err
echo "bench rc=$?" >> gpurun_out/r3ncu3/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3ncu3/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-mlp --no-schedule --no-e2e > gpurun_out/r3ncu3/ncu_launch.log 2>&1
echo "launch list rc=$?" >> gpurun_out/r3ncu3/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ssp_rkey_kernel -o gpurun_out/r3ncu3/rkey_full python tools/ssp_one.py 10000 1 > gpurun_out/r3ncu3/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/r3ncu3/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_exact_kernel -c 1 -o gpurun_out/r3ncu3/score_full python tools/ssp_one.py 10000 1 > gpurun_out/r3ncu3/ncu_score.log 2>&1
echo "score rc=$?" >> gpurun_out/r3ncu3/status.txt
MUX_VERBOSE=1 timeout 120 python tools/ssp_one.py 10000 2 > gpurun_out/r3ncu3/levels.log 2>&1
echo "levels rc=$?" >> gpurun_out/r3ncu3/status.txt
