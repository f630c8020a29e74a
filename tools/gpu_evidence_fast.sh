#!/bin/bash
# Evidence pass without the test suite: default bench line, ncu launch list, one full capture of k_rqi_fb.
# usage: gpurun --timeout 2400 -- 'bash tools/gpu_evidence_fast.sh <tag>'
set -u
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${TAG}_smi.txt 2>&1
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench exit $?" >> $O/${TAG}_bench.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --other-configs= --emulate-world= --no-zstore --dense="
timeout 600 $CMD > $O/${TAG}_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $O/${TAG}_launches.csv $CMD > $O/${TAG}_ncu_launch.log 2>&1
echo "launch-list exit $?" >> $O/${TAG}_ncu_launch.log
PC="python tools/prof_case.py 5 2"
timeout 300 $PC > $O/${TAG}_case.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:^k_rqi_fb -s 1 -c 1 \
    -o $O/${TAG}_rqi_fb_full -f $PC > $O/${TAG}_ncu.log 2>&1
echo "exit $?" >> $O/${TAG}_ncu.log
