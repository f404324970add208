#!/bin/bash
# usage: gpurun -- bash tools/gpu_round2.sh TAG
TAG=${1:-run}
mkdir -p gpurun_out
python -c "from oracle import cproj; cproj.build()"
timeout 1200 python -m pytest tests/test_gpu_scale.py -q -s -k "tensor_pipe" > gpurun_out/${TAG}_tc_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_tc_tests.log
bash tools/gpu_bench.sh ${TAG}_tc "c5shard c3" --steps 3 --warmup 3 --order tc --no-cpu-baseline
# launch list of the default bench command (C2): after the plain run above exits 0
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_c2_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 9000 --csv --log-file gpurun_out/${TAG}_c2_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_c2_ncu.log 2>&1
if [ -d oracle/_ref/conformance ]; then bash tools/conformance.sh run ${TAG}; fi
tail -3 gpurun_out/${TAG}*.log
