#!/bin/bash
# Round-2 evidence pass: GPU tests, default bench line, ncu launch list of the bench command.
# usage: gpurun --timeout 3600 -- 'bash tools/gpu_evidence_r02.sh <tag>'
set -u
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${TAG}_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > $O/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest.log
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench exit $?" >> $O/${TAG}_bench.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --other-configs= --emulate-world= --no-zstore --dense="
timeout 600 $CMD > $O/${TAG}_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $O/${TAG}_launches.csv $CMD > $O/${TAG}_ncu_launch.log 2>&1
echo "launch-list exit $?" >> $O/${TAG}_ncu_launch.log
