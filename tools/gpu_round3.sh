#!/bin/bash
# usage: gpurun -- bash tools/gpu_round3.sh TAG
TAG=${1:-run}
mkdir -p gpurun_out
python -c "from oracle import cproj; cproj.build()"
timeout 1500 python -m pytest tests/test_gpu_scale.py -q -s -k "tensor_pipe or reduced" > gpurun_out/${TAG}_tc_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_tc_tests.log
for d in 6 4 3; do
  timeout 900 python bench.py --config c5shard --steps 3 --warmup 3 --order tc --sketch-digits $d --no-cpu-baseline > gpurun_out/${TAG}_c5_tc_d$d.json 2> gpurun_out/${TAG}_c5_tc_d$d.err
done
if [ -d oracle/_ref/conformance ]; then bash tools/conformance.sh run ${TAG}; fi
grep -E "passed|failed" gpurun_out/${TAG}*.log
