#!/bin/bash
# NEXT-1b / NEXT-3 checks: their GPU tests, then an A/B of MR3_RELAX on the given configs
set -u
O=gpurun_out; mkdir -p $O
TAG=${1:-next}
shift || true
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "relaxed_isolation or absolute_gap or backtracking or rare_paths or glued or config1 or fp32" > $O/${TAG}_pytest.log 2>&1; echo "pytest exit $?" >> $O/${TAG}_pytest.log
bash tools/gpu_ab.sh $TAG RELAX 0 0.5 "$@"
