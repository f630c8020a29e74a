#!/bin/bash
# Final pass of a session: FP64/other-pipe issue microbenchmark, the default bench line, the GPU test suite.
# usage: gpurun --timeout 3000 -- 'bash tools/gpu_final.sh <tag>'
set -u
TAG=${1:-fin}
O=gpurun_out
mkdir -p $O
timeout 120 ./tools/micro/fp64mix > $O/${TAG}_fp64mix.txt 2>&1
echo "fp64mix exit $?" >> $O/${TAG}_fp64mix.txt
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench exit $?" >> $O/${TAG}_bench.err
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > $O/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest.log
