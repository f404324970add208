#!/bin/bash
# One gpurun call: full GPU suite + smoke + the bench lines of every config.
# usage: gpurun -- bash tools/gpu_round.sh TAG
TAG=${1:-run}
mkdir -p gpurun_out
bash tools/gpu_tests.sh $TAG
bash tools/gpu_bench.sh $TAG "c2" --steps 10 --warmup 3
bash tools/gpu_bench.sh ${TAG}_tc "c5shard" --steps 3 --warmup 3 --order tc --no-cpu-baseline
bash tools/gpu_bench.sh ${TAG}_ref "c5shard" --steps 3 --warmup 3 --order reference --no-cpu-baseline
bash tools/gpu_bench.sh ${TAG} "c3 c1 c4" --steps 3 --warmup 3 --no-cpu-baseline
bash tools/gpu_bench.sh ${TAG}_l2 "c2" --steps 5 --warmup 3 --interblock l2_plus_cholqr --no-cpu-baseline --no-e2e
tail -3 gpurun_out/${TAG}*_bench_*.err
