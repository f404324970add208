#!/bin/bash
# compute-sanitizer record of the warp-specialised kernels:
#   gpurun -- bash tools/sanitize.sh TAG
TAG=${1:-san}
mkdir -p gpurun_out
timeout 300 python tools/sanitize_case.py > gpurun_out/${TAG}_plain.log 2>&1 || exit 1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py > gpurun_out/${TAG}_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_$tool.log
  tail -4 gpurun_out/${TAG}_$tool.log
done
