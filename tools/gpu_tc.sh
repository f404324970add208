#!/bin/bash
# usage: gpurun -- bash tools/gpu_tc.sh TAG
TAG=${1:-tc}
mkdir -p gpurun_out
timeout 300 python tools/tc_probe.py check > gpurun_out/${TAG}_check.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_check.log
if grep -q "ALL OK" gpurun_out/${TAG}_check.log; then
  timeout 600 python tools/tc_probe.py time > gpurun_out/${TAG}_time.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_time.log
  python -c "from oracle import cproj; cproj.build()"
  timeout 900 python -m pytest tests/test_gpu_scale.py -q -s -k "tensor_pipe or tc" > gpurun_out/${TAG}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_tests.log
fi
cat gpurun_out/${TAG}_check.log gpurun_out/${TAG}_time.log
