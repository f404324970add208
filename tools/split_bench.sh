mkdir -p gpurun_out
for v in "SPLIT_BENCH_LIB=tools/_base/librbgs_b200.so" "RB_X=1" "SPLIT_BENCH_LIB=tools/_base/librbgs_b200.so" "RB_X=2"; do
  env $v timeout 300 python tools/split_bench.py >> gpurun_out/split_bench.jsonl 2>> gpurun_out/split_bench.err
done
