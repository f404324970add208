mkdir -p gpurun_out
for v in "RB_SPLIT_MODE=1" "RB_SPLIT_MODE=2"; do
  env $v timeout 300 python tools/split_bench.py >> gpurun_out/split_bench.jsonl 2>> gpurun_out/split_bench.err
done
