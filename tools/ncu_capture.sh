#!/bin/bash
# Dev: ncu captures of the step's kernels on the GPU box, summarised there (the .ncu-rep files
# are too large to bring back through gpurun_out).  Usage: tools/ncu_capture.sh TAG CFG
set -u
TAG=${1:-r02}; CFG=${2:-cfg4}
OUT=gpurun_out
REP=/tmp/${TAG}_full_${CFG}
ncu --set full --clock-control none --import-source on \
    -k regex:"k_onesweep|k_lsd_count|k_proj_tc|k_finalize|k_query_lat|k_brute8|k_gram_fused" -c 24 \
    -o $REP -f python tools/ncu_driver.py $CFG > $OUT/${TAG}_ncu_full_${CFG}.log 2>&1
python tools/tools_ncu_summary.py $REP.ncu-rep > $OUT/${TAG}_ncu_full_${CFG}.txt 2>&1
python tools/ncu_traffic.py $REP.ncu-rep $CFG --out $OUT/${TAG}_traffic_${CFG}.json > /dev/null 2>&1
ncu -i $REP.ncu-rep --page details --csv > $OUT/${TAG}_ncu_details_${CFG}.csv 2>/dev/null
ls -la $REP.ncu-rep >> $OUT/${TAG}_ncu_full_${CFG}.log
