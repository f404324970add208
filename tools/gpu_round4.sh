#!/bin/bash
TAG=${1:-run}
mkdir -p gpurun_out
python -c "from oracle import cproj; cproj.build()"
timeout 2400 python -m pytest tests -m gpu -q --deselect tests/test_gpu_scale.py -x > gpurun_out/${TAG}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_tests.log
if [ -d oracle/_ref/conformance ]; then bash tools/conformance.sh run ${TAG}; fi
grep -E "passed|failed" gpurun_out/${TAG}*.log
