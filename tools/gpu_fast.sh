#!/bin/bash
# Fast iteration pass: a parity subset, all-configs timing, config-5 bench line (no e2e/cpu/emulation).
# usage: gpurun --timeout 1500 -- 'bash tools/gpu_fast.sh <tag> [pytest -k expr|none]'
set -u
TAG=${1:-f}
SEL=${2:-"rqi_fb_matches or newton_path or config1 or small_random_full or glued_wilkinson_small or fp32_subset"}
O=gpurun_out
mkdir -p $O
if [ "$SEL" != "none" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -k "$SEL" > $O/${TAG}_pytest.log 2>&1
  echo "pytest exit $?" >> $O/${TAG}_pytest.log
fi
timeout 300 python tools/all_configs.py > $O/${TAG}_configs.log 2>&1
echo "configs exit $?" >> $O/${TAG}_configs.log
timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --other-configs= --emulate-world= --no-zstore \
    > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench exit $?" >> $O/${TAG}_bench.err
