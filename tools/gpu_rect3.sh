#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
MUX_VERBOSE=0 timeout 900 python tools/rect_check.py > gpurun_out/rect_check.log 2> gpurun_out/rect_check.err
timeout 600 python -m pytest tests/test_gpu_ssp.py -q -x > gpurun_out/pytest_ssp.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_ssp.log
echo finished
