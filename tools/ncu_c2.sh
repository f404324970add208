# ncu evidence for the C2 bench command (run on the GPU box from the repo root):
# launch list + one --set full capture each of the sketch, its pre-pass and
# the projection; reports stay in /tmp, summaries go to gpurun_out/.
set -x
O=gpurun_out/ncu; R=/tmp/ncu; mkdir -p $O $R
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $R/launches.csv $B > $O/list.log 2>&1; echo list=$?
python tools/launch_summary.py $R/launches.csv > $O/launches.txt
gzip -c $R/launches.csv > $O/launches.csv.gz
for spec in "gauss_tc_partial 10" "encode_planes 10" "chunk_max 10" "sumsq3_kernel 10"; do
  set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:$1 --launch-skip $2 -c 1 -o $R/$1 $B > $O/$1.log 2>&1; echo $1=$?
  python tools/ncu_summary.py $R/$1.ncu-rep > $O/$1.json
  ncu -i $R/$1.ncu-rep --page raw --csv > $O/$1_raw.csv
  ncu -i $R/$1.ncu-rep --page source --csv 2>/dev/null | gzip -c > $O/$1_source.csv.gz
done
du -sh $O
