#!/bin/bash
# Quick pass: GPU tests (optionally filtered) and one bench line.
# usage: gpurun --timeout 1800 -- 'bash tools/gpu_quick.sh <tag> [pytest -k expr|all|none]'
set -u
TAG=${1:-q}
SEL=${2:-all}
O=gpurun_out
mkdir -p $O
if [ "$SEL" != "none" ]; then
  if [ "$SEL" = "all" ]; then
    timeout 2400 python -m pytest tests -m gpu -q -x --durations=30 > $O/${TAG}_pytest.log 2>&1
  else
    timeout 1500 python -m pytest tests -m gpu -q -x -k "$SEL" > $O/${TAG}_pytest.log 2>&1
  fi
  echo "pytest exit $?" >> $O/${TAG}_pytest.log
fi
timeout 600 python bench.py --steps 5 --warmup 3 > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench exit $?" >> $O/${TAG}_bench.err
