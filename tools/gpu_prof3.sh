#!/bin/bash
# ncu --set full capture (config 5, second solve) of one kernel; exports raw + sass-source CSV
# and removes the report (gpurun copies back <= 64 MiB).  usage: gpu_prof3.sh <tag> <kernel> [skip]
O=gpurun_out; TAG=${1:-p3}; K=${2:-k_rqi}; SKIP=${3:-1}
CMD="python tools/prof_case.py 5 2"
timeout 300 $CMD > $O/${TAG}_case.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:^${K}$ -s $SKIP -c 1 \
    -o /tmp/${TAG}_${K} -f $CMD > $O/${TAG}_ncu_${K}.log 2>&1
echo "exit $?" >> $O/${TAG}_ncu_${K}.log
ncu -i /tmp/${TAG}_${K}.ncu-rep --page raw --csv > $O/${TAG}_${K}_raw.csv 2>/dev/null
ncu -i /tmp/${TAG}_${K}.ncu-rep --page source --csv --print-source sass > $O/${TAG}_${K}_sass.csv 2>/dev/null
ls -la /tmp/${TAG}_${K}.ncu-rep >> $O/${TAG}_ncu_${K}.log 2>&1
