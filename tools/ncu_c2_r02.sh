# Round-2 ncu evidence for the C2 bench command (run on the GPU box from the
# repo root, AFTER the plain command exited 0): launch list + one --set full
# capture each of the projection, the sketch, its pre-pass and the
# k-dimensional kernels; summaries (pipe-cycle metrics, clocks) to gpurun_out/.
O=gpurun_out/ncu_r02; R=/tmp/ncu_r02; mkdir -p $O $R
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$B > $O/plain.json 2> $O/plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $R/launches.csv $B > $O/list.log 2>&1; echo list=$?
python tools/launch_summary.py $R/launches.csv > $O/launches.txt
gzip -c $R/launches.csv > $O/launches.csv.gz
for spec in "project_staged 12" "gauss_tc_partial 12" "encode_tile 12" "chunk_max 12" "richardson_v4 12" "cholqr_v4 12" "certify_coop 0"; do
  set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:$1 --launch-skip $2 -c 1 -f -o $R/$1 $B > $O/$1.log 2>&1; echo $1=$?
  python tools/ncu_summary.py $R/$1.ncu-rep > $O/$1.json
done
ls -la $O
