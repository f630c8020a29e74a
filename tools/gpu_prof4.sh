#!/bin/bash
# ncu --set full capture of one kernel on a config (second solve); exports raw + SASS source
# CSV.  usage: gpu_prof4.sh <tag> <kernel regex> <config> [il iu]
O=gpurun_out; TAG=$1; K=$2; CFG=$3; shift 3
CMD="python tools/prof_case.py $CFG 2 $*"
timeout 300 $CMD > $O/${TAG}_case.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:${K} -s 1 -c 1 \
    -o /tmp/${TAG} -f $CMD > $O/${TAG}_ncu.log 2>&1
echo "exit $?" >> $O/${TAG}_ncu.log
ncu -i /tmp/${TAG}.ncu-rep --page raw --csv > $O/${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/${TAG}.ncu-rep --page source --csv --print-source sass > $O/${TAG}_sass.csv 2>/dev/null
gzip -f $O/${TAG}_sass.csv
ls -la /tmp/${TAG}.ncu-rep >> $O/${TAG}_ncu.log 2>&1
