#!/bin/bash
# full-size (config 5, all 50000 eigenvalues, values only) ncu capture of k_bisect_s and k_rqi_locate
O=gpurun_out; TAG=${1:-pb}
CMD="python tools/prof_case.py 5 2 1 50000 N"
timeout 300 $CMD > $O/${TAG}_case.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^k_bisect_s$ -s 1 -c 1 \
    -o $O/${TAG}_bisect_full -f $CMD > $O/${TAG}_ncu.log 2>&1
echo "exit $?" >> $O/${TAG}_ncu.log
