#!/bin/bash
# Evidence pass: bench line, ncu launch list of the bench command, ncu --set full of the
# top kernels (CSV exports; reports removed so gpurun_out stays < 64 MiB).
# usage: gpurun --timeout 3600 -- 'bash tools/gpu_evidence.sh <tag>'
set -u
TAG=${1:-ev}
O=gpurun_out
mkdir -p $O
timeout 600 python bench.py --steps 8 --warmup 3 > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench exit $?" >> $O/${TAG}_bench.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 $CMD > $O/${TAG}_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
    --log-file $O/${TAG}_launches.csv $CMD > $O/${TAG}_ncu_launch.log 2>&1
echo "launch-list exit $?" >> $O/${TAG}_ncu_launch.log
bash tools/gpu_prof3.sh ${TAG} k_rqi 1
bash tools/gpu_prof3.sh ${TAG} k_bisect_s 1
bash tools/gpu_prof3.sh ${TAG} k_rqi_locate 1
bash tools/gpu_prof3.sh ${TAG} k_cell_counts 3
rm -f $O/${TAG}_*_sass.csv.gz
for f in $O/${TAG}_*_sass.csv; do gzip -f $f; done
