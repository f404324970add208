#!/bin/bash
TAG=${1:-run}
mkdir -p gpurun_out
python -c "from oracle import cproj; cproj.build()"
timeout 1500 python -m pytest tests/test_gpu_scale.py -q -s -k "tensor_pipe or reduced" > gpurun_out/${TAG}_tc_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_tc_tests.log
timeout 900 python bench.py --config c5shard --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err
timeout 600 python bench.py --config c3 --order tc --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c3tc.json 2> gpurun_out/${TAG}_c3tc.err
grep -E "passed|failed" gpurun_out/${TAG}*.log
