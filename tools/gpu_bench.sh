#!/bin/bash
# usage: gpurun -- bash tools/gpu_bench.sh TAG "c2 c3 c5shard c1 c4" [extra bench args]
TAG=${1:-run}
CFGS=${2:-c2}
shift 2
mkdir -p gpurun_out
for c in $CFGS; do
  timeout 900 python bench.py --config $c "$@" > gpurun_out/${TAG}_bench_${c}.json 2> gpurun_out/${TAG}_bench_${c}.err
  echo "bench $c rc=$?" >> gpurun_out/${TAG}_bench_${c}.err
done
