#!/bin/bash
# Full evidence pass: GPU tests, bench line, ncu launch list of the bench command,
# ncu --set full of the full-size k_rqi and k_bisect_s launches (config 5).
# usage: gpurun --timeout 3600 -- 'bash tools/gpu_full.sh <tag>'
set -u
TAG=${1:-full}
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench exit $?" >> $O/${TAG}_bench.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 $CMD > $O/${TAG}_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $O/${TAG}_launches.csv $CMD > $O/${TAG}_ncu_launch.log 2>&1
echo "launch-list exit $?" >> $O/${TAG}_ncu_launch.log
CMD2="python tools/prof_case.py 5 2"
timeout 300 $CMD2 > $O/${TAG}_case.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:^k_rqi$ -s 1 -c 1 \
    -o $O/${TAG}_rqi -f $CMD2 > $O/${TAG}_ncu_rqi.log 2>&1
echo "ncu rqi exit $?" >> $O/${TAG}_ncu_rqi.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:^k_bisect_s$ -s 2 -c 1 \
    -o $O/${TAG}_bisect -f $CMD2 > $O/${TAG}_ncu_bisect.log 2>&1
echo "ncu bisect exit $?" >> $O/${TAG}_ncu_bisect.log
