#!/bin/bash
# debug helper: run the sparse-sign sketch cases under compute-sanitizer
CS=/usr/local/cuda/bin/compute-sanitizer
ls -la $CS 2>&1 | head -1
for c in "5000 120 8 0 5" "1024 64 3 0 4" "3001 488 8 7 9" "2500 40 16 2048 1"; do
  for pth in 0 1; do
    CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/sp_dbg.py $c $pth > gpurun_out/o_$pth.txt 2>&1
    echo "--- $c $pth rc=$?"
    grep -E "^ok|table ok|Invalid|at 0x|by thread|rror" gpurun_out/o_$pth.txt | head -8
  done
done
