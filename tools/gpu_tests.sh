#!/bin/bash
# One gpurun call: build check, new scale tests, the full GPU suite, smoke.
# usage: gpurun -- bash tools/gpu_tests.sh TAG [pytest -k expr]
TAG=${1:-run}
K=${2:-}
mkdir -p gpurun_out
python -c "from oracle import cproj; cproj.build()" > gpurun_out/${TAG}_cproj.log 2>&1
if [ -n "$K" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -k "$K" -s > gpurun_out/${TAG}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_tests.log
else
  timeout 1500 python -m pytest tests/test_gpu_scale.py -q -s > gpurun_out/${TAG}_scale.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_scale.log
  timeout 2400 python -m pytest tests -m gpu -q --deselect tests/test_gpu_scale.py > gpurun_out/${TAG}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_tests.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
fi
tail -5 gpurun_out/${TAG}_*.log
