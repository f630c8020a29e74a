#!/bin/bash
# Iteration pass: GPU tests, bench line, ncu --set full of k_rqi (config-5 subset) and k_bisect.
# usage: gpurun --timeout 2400 -- 'bash tools/gpu_iter.sh <tag> [notests]'
set -u
TAG=${1:-it}
O=gpurun_out
mkdir -p $O
if [ "${2:-}" != "notests" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest.log 2>&1
  echo "pytest exit $?" >> $O/${TAG}_pytest.log
fi
timeout 600 python bench.py --steps 3 --warmup 3 > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench exit $?" >> $O/${TAG}_bench.err
CMD="python tools/prof_case.py 5 2 20001 28192"
timeout 300 $CMD > $O/${TAG}_case.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^k_rqi$ -s 1 -c 1 \
    -o $O/${TAG}_rqi -f $CMD > $O/${TAG}_ncu_rqi.log 2>&1
echo "ncu rqi exit $?" >> $O/${TAG}_ncu_rqi.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^k_bisect_s$ -s 1 -c 1 \
    -o $O/${TAG}_bisect -f $CMD > $O/${TAG}_ncu_bisect.log 2>&1
echo "ncu bisect exit $?" >> $O/${TAG}_ncu_bisect.log
