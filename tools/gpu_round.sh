#!/bin/bash
# One GPU-box pass: parity tests, bench line, ncu launch list, ncu --set full of k_bisect.
# usage (from this container): gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [tag]'
set -u
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${TAG}_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench exit $?" >> $O/${TAG}_bench.err
# launch list of the same command line (run once plain first, then under ncu)
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 600 $CMD > $O/${TAG}_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/${TAG}_launches.csv $CMD > $O/${TAG}_ncu_launch.log 2>&1
echo "launch-list exit $?" >> $O/${TAG}_ncu_launch.log
# full section set of the dominant kernel (last warm-up's k_bisect launch)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_bisect -s 2 -c 1 \
    -o $O/${TAG}_bisect -f $CMD > $O/${TAG}_ncu_full.log 2>&1
echo "ncu full exit $?" >> $O/${TAG}_ncu_full.log
