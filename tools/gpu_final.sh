#!/bin/bash
# Final round-2 GPU pass: every GPU test, smoke, the bench lines of every config.
TAG=${1:-r02_final}
mkdir -p gpurun_out
python -c "from oracle import cproj; cproj.build()"
timeout 2400 python -m pytest tests/test_gpu_scale.py -q -s > gpurun_out/${TAG}_scale.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_scale.log
timeout 2400 python -m pytest tests -m gpu -q --deselect tests/test_gpu_scale.py > gpurun_out/${TAG}_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
timeout 900 python bench.py --config c5shard --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_c5shard.json 2> gpurun_out/${TAG}_bench_c5shard.err
timeout 900 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err
timeout 900 python bench.py --config c3 --order tc --steps 3 --warmup 3 --no-e2e > gpurun_out/${TAG}_bench_c3_tc.json 2> gpurun_out/${TAG}_bench_c3_tc.err
timeout 900 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_c1.json 2> gpurun_out/${TAG}_bench_c1.err
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --diagnostics sketched > gpurun_out/${TAG}_bench_c4_sketched.json 2> gpurun_out/${TAG}_bench_c4_sketched.err
grep -E "passed|failed|smoke" gpurun_out/${TAG}_*.log
