#!/bin/bash
# full-size (config 5, all 50000 eigenpairs) ncu capture of k_rqi (replay saves/restores Z)
O=gpurun_out; TAG=${1:-pr}
CMD="python tools/prof_case.py 5 2"
timeout 300 $CMD > $O/${TAG}_case.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:^k_rqi$ -s 1 -c 1 \
    -o $O/${TAG}_rqi_full -f $CMD > $O/${TAG}_ncu.log 2>&1
echo "exit $?" >> $O/${TAG}_ncu.log
