#!/bin/bash
TAG=${1:-run}
mkdir -p gpurun_out
timeout 900 python bench.py --config c5shard --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_c5shard.json 2> gpurun_out/${TAG}_bench_c5shard.err
timeout 900 python bench.py --config c3 --order tc --steps 3 --warmup 3 --no-e2e > gpurun_out/${TAG}_bench_c3_tc.json 2> gpurun_out/${TAG}_bench_c3_tc.err
for m in tensor tensor4 tensor3; do
  SB_N=16777216 SB_P=64 SB_K=2048 SB_MODE=$m timeout 600 python tools/split_bench.py > gpurun_out/${TAG}_split_c5_$m.json 2>&1
done
python tools/tc_probe.py one 16777216 64 512 && ncu --set full --clock-control none --import-source on -k regex:project_tc2 -c 1 -s 2 -o gpurun_out/${TAG}_tc2_c5 -f python tools/tc_probe.py one 16777216 64 512 > gpurun_out/${TAG}_ncu_tc2.log 2>&1
SB_N=16777216 SB_P=64 SB_K=2048 SB_MODE=tensor4 ncu --set full --clock-control none --import-source on -k regex:gauss_tc_partial -c 1 -s 3 -o gpurun_out/${TAG}_gauss_d4_c5 -f python tools/split_bench.py > gpurun_out/${TAG}_ncu_gauss.log 2>&1
cat gpurun_out/${TAG}_split_c5_*.json | cut -c1-500
