# one --set full capture of the C5-shard gaussian sketch (NP = 64 pair launch)
O=gpurun_out/ncu5; R=/tmp/ncu5; mkdir -p $O $R
B="python bench.py --config c5shard --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:gauss_tc_partial --launch-skip 6 -c 1 -o $R/g $B > $O/g.log 2>&1; echo g=$?
python tools/ncu_summary.py $R/g.ncu-rep > $O/gauss_c5.json
ncu -i $R/g.ncu-rep --page source --csv 2>/dev/null | gzip -c > $O/gauss_c5_source.csv.gz
