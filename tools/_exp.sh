for rep in 1 2; do
for mode in 2 3; do
  echo "== split mode $mode tensor4 C5"; RB_SPLIT_MODE=$mode SB_N=16777216 SB_P=64 SB_K=2048 SB_MODE=tensor4 python tools/split_bench.py 2>/dev/null | tail -1 | cut -c60-330
done
done
for mode in 2 3; do
  echo "== split mode $mode tensor C2"; RB_SPLIT_MODE=$mode python tools/split_bench.py 2>/dev/null | tail -1 | cut -c60-330
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv
