#!/bin/bash
TAG=${1:-run}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kdim.py -q -k "gemm or syrk" > gpurun_out/${TAG}_kdim_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_kdim_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "gmres or arnoldi" > gpurun_out/${TAG}_gmres_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_gmres_tests.log
timeout 600 python bench.py --config c4 --steps 2 --warmup 2 > gpurun_out/${TAG}_c4_full.json 2> gpurun_out/${TAG}_c4_full.err
timeout 600 python bench.py --config c4 --steps 2 --warmup 2 --diagnostics sketched > gpurun_out/${TAG}_c4_sketched.json 2> gpurun_out/${TAG}_c4_sketched.err
grep -E "passed|failed" gpurun_out/${TAG}*.log; cat gpurun_out/${TAG}_c4_*.json | cut -c1-400
