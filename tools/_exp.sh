for cfg in "4096 512 1 1" "4096 1024 1 1"; do
  set -- $cfg
  echo "== LBO=$1 SBO=$2 LAYOUT=$3 AMAJOR=$4"
  RB_TC_DEBUG=1 RB_TC_LBO=$1 RB_TC_SBO=$2 RB_TC_LAYOUT=$3 RB_TC_AMAJOR=$4 timeout 60 python tools/tc_probe.py map 2>&1 | grep -E "raw k|acc row|mismatches|out\[|rror" | head -50
done
timeout 200 python tools/tc_probe.py check 2>&1 | tail -12
